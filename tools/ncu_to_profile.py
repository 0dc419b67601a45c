"""Turn a gpurun ncu capture into the committed profile summaries under profiles/:
    python tools/ncu_to_profile.py gpurun_out/TAG_cfg2.ncu-rep profiles/r1_TAG_cfg2_ncu_full.csv [cfg]
writes the key metrics (duration, DRAM bytes, issue / pipe utilisation, occupancy, stalls) and
updates profiles/ncu_traffic.json with the DRAM bytes per launch for bench.py's roofline."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "smsp__cycles_active.avg", "sm__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warp_latency_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_sample_count"]


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    vals = dict(zip(h, v))
    unit = dict(zip(h, units))
    with open(dst, "w") as f:
        f.write(f"# ncu --set full --clock-control none, kernel {vals.get('Kernel Name', '?')[:120]}\n")
        f.write(f"# source report: {os.path.basename(rep)} (gpurun_out, not committed)\n")
        f.write("metric,unit,value\n")
        for k in KEYS:
            if k in vals:
                f.write(f"{k},{unit.get(k, '')},{vals[k]}\n")
    def num(k):
        x = vals.get(k, "0").replace(",", "")
        return float(x) if x else 0.0
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = num("dram__bytes_read.sum") * scale.get(unit.get("dram__bytes_read.sum", "byte"), 1) + \
        num("dram__bytes_write.sum") * scale.get(unit.get("dram__bytes_write.sum", "byte"), 1)
    tj = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d[cfg] = {"dram_bytes_per_launch": dram, "source": os.path.basename(dst)}
    json.dump(d, open(tj, "w"), indent=1)
    print(f"wrote {dst}; DRAM bytes per launch {dram:.4g}")


if __name__ == "__main__":
    main()
