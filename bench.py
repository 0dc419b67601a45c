#!/usr/bin/env python3
"""Benchmark of the B200 joint-acceleration bilateral filter (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

A "step" is one bf_apply of the whole hot path (modulate + box sums + combine + divide) over one
synthetic image of the workload (BASELINE.json configs; default cfg2 = 4096x4096 f32, the config
the north_star target is quoted on). Inputs are resident in HBM before the timed region; L2 is
flushed (a 256 MiB write) before every timed step and the step is timed alone with CUDA events
on the launching stream. For N > 1 (torchrun) every rank filters its own image (independent
problems, weak scaling), times are max-reduced over ranks, value = all ranks' pixels / max time.
`e2e` repeats the metric through bf_apply_host (pinned host input -> device -> host output).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/sec per grayscale BF at given sigma_s, sigma_r, N; % of HBM roofline"
UNIT = "MP/s"


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0,
            "_source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """Samples SM clocks and clock-event (throttle) reasons while the timed region runs: NVML every
    20 ms (nvidia_ml_py), else nvidia-smi every 200 ms."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []      # (sm_mhz, max_mhz, power_w, reasons bitmask)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml:
            nv, h = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            return (float(sm), float(mx), pw, int(rs))
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        c = [x.strip() for x in out.stdout.strip().split(",")]
        mask = sum(bit for bit, v in zip((0x8, 0x40, 0x20, 0x4), c[3:7]) if v.lower() == "active")
        return (float(c[0]), float(c[1]), float(c[2]) if c[2].replace(".", "").isdigit() else 0.0, mask)

    def _loop(self):
        period = 0.02 if self._nvml else 0.2
        while not self._stop.is_set():
            try:
                self.rows.append(self._sample())
            except Exception:
                pass
            self._stop.wait(period)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        reasons = sorted({n for r in self.rows for n, bit in self.NAMES.items() if r[3] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(r[2] for r in self.rows),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if os.environ.get("BF_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        dist.init_process_group(backend)
    return world, rank, local


def reduce_max(x: float, world: int, device=None) -> float:
    """max over ranks (device timing is max-reduced; never wall clock)."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def config_dict(spec, flush: bool, world: int) -> dict:
    return {"workload": f"{spec.name}: {spec.H}x{spec.W} {'uint8' if spec.gen == 'ramp' and not spec.as_f32 else 'float32'}"
                        f" {spec.gen}, K_s {spec.spatial} sigma_s={spec.sigma_s} r={spec.radius}, "
                        f"K_r {spec.range_kind} sigma_r={spec.sigma_r}, N={spec.n_terms}, D={spec.intensity_max}",
            "H": spec.H, "W": spec.W, "frames_per_step": 1, "n_spatial": 9,
            "l2": "flushed (256 MiB write) before every timed step" if flush else "not flushed",
            "parallelism": f"dp{world} (independent images per rank)" if world > 1 else "single GPU"}


# --------------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands (TEST INFRASTRUCTURE used only here and in tests)
# --------------------------------------------------------------------------------------------

def oracle_sample_rate(spec, side: int) -> tuple:
    """Time the oracle (fp64 numpy SAT evaluation) on a side x side crop of the workload."""
    from oracle import bf as obf
    from oracle import fit as ofit
    from synth import config_input, config_params
    full = config_input(spec, H=min(spec.H, 1024), W=min(spec.W, 1024))
    crop = full[:side, :side]
    plan = ofit.make_plan(**config_params(spec))
    t0 = time.perf_counter()
    obf.bf_box(crop, plan)
    dt = time.perf_counter() - t0
    return crop.size / dt / 1e6, dt, f"{side}x{side} crop of the {spec.name} input, full oracle (fp64 SAT evaluation)"


def run_reference(args, spec):
    world, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return 0
    side = args.ref_side
    rates = []
    samples = []
    for i in range(args.warmup + args.steps):
        r, dt, desc = oracle_sample_rate(spec, side)
        if i >= args.warmup:
            rates.append(r)
            samples.append(dt)
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(samples),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(spec, False, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "single-process numpy fp64 oracle on the GPU box's host cores; each step is a bounded sample"}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------

def traffic_per_launch(cfg: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(cfg, {}).get("dram_bytes_per_launch")


def run_ours(args, spec):
    import torch
    from paper_1803_00004_b200 import build
    build.build()
    import paper_1803_00004_b200 as bfp
    from synth import config_input

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    u8 = (spec.gen == "ramp" and not spec.as_f32)
    plan = bfp.Plan(spatial=spec.spatial, range_kind=spec.range_kind, sigma_s=spec.sigma_s, sigma_r=spec.sigma_r,
                    radius=spec.radius, n_terms=spec.n_terms, intensity_max=spec.intensity_max,
                    input_dtype="u8" if u8 else "f32")
    img_np = config_input(spec)
    img = torch.from_numpy(img_np).to(dev)
    out = torch.empty(img.shape, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    H, W = img.shape
    launches = bfp.launches(plan, H, W)     # kernel launches per bf_apply (bf_apply_launches)
    lcfg = bfp.config(plan, H, W)            # the kernel and launch shape bf_apply enqueues (bf_apply_config)

    def step():
        bfp.apply(plan, img.data_ptr(), out.data_ptr(), H, W, sptr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    times = []
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier(world)
    total_ms = reduce_max(sum(times), world, dev)
    ms = total_ms / args.steps
    mpix_all = world * H * W * args.steps / 1e6
    value = mpix_all / (total_ms / 1e3)

    # ---- end to end through the public host API (pinned host buffers, copies inside the timing)
    h_in = torch.from_numpy(img_np).pin_memory()
    h_out = torch.empty((H, W), dtype=torch.float32).pin_memory()
    for _ in range(max(1, args.warmup // 2)):
        bfp.apply_host(plan, h_in.data_ptr(), h_out.data_ptr(), H, W, sptr)
    barrier(world)
    e2e_t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        bfp.apply_host(plan, h_in.data_ptr(), h_out.data_ptr(), H, W, sptr)
        e2e_t.append(time.perf_counter() - t0)
    e2e_total = reduce_max(sum(e2e_t), world, dev)
    e2e_value = world * H * W * args.steps / 1e6 / e2e_total

    if rank != 0:
        barrier(world)
        return 0
    peaks = measured_peaks()
    bytes_per_px = (1 if u8 else 4) + 4
    alg_bytes = H * W * bytes_per_px
    hbm_gbs = alg_bytes / (ms / 1e3) / 1e9
    hbm_peak = float(peaks["hbm_gbs"])
    clocks = sampler.summary()
    nk = len(plan.info()["k"])
    C = 4 * nk
    # ALU roofline (the bound of this path): SURVEY 8(d)'s algorithmic work of
    # >= 8 FP32-lane ops per box-filtered channel per pixel, against 148 SMs x 128 FP32 lanes x the
    # SM clock measured under load (max clock if nvidia-smi gave none)
    sm_mhz = clocks.get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e12                  # T lane-op/s
    alu_ops = 8.0 * C * H * W                                    # per step
    alu_achieved = alu_ops / (ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 channels, i32 box sums, i64 combine", "data": "synthetic",
        "config": config_dict(spec, True, world),
        "roofline": {"bound": "alu", "achieved": alu_achieved, "peak": alu_peak, "unit": "T lane-op/s",
                     "frac": alu_achieved / alu_peak, "traffic": traffic_per_launch(spec.name),
                     "kernel": lcfg["kernel"], "launches_per_step": launches,
                     "launch": {"threads_per_cta": lcfg["threads_per_cta"], "grid": list(lcfg["grid"]),
                                "tile": list(lcfg["tile"]), "smem_bytes": lcfg["smem_bytes"]},
                     "algorithmic_ops_per_step": alu_ops,
                     "peak_source": f"148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (B200_PROFILING.md unit counts)",
                     "note": "SURVEY 8(d): >= 8 FP32-lane ops per channel-pixel, C = 4 N_eff channels"},
        "hbm_roofline": {"achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_gbs / hbm_peak,
                         "algorithmic_bytes_per_step": alg_bytes,
                         "peak_source": peaks["_source"] + " hbm_gbs",
                         "note": "BASELINE metric: image bytes in + out at the measured HBM bandwidth"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(img_np.nbytes),
                "d2h_bytes_per_step": int(H * W * 4)},
        "gpu_launches": args.steps * launches,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline:
        r, dt, desc = oracle_sample_rate(spec, args.ref_side)
        line["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                                "seconds": dt}
    print(json.dumps(line), flush=True)
    barrier(world)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-side", type=int, default=768, help="side of the oracle's timed crop")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    from synth import CONFIGS
    spec = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, spec)
    return run_ours(args, spec)


if __name__ == "__main__":
    sys.exit(main())
