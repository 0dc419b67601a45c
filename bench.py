#!/usr/bin/env python3
"""Benchmark of the B200 joint-acceleration bilateral filter (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
                    [--n-spatial 9] [--no-per-config] [--no-cpu-baseline]

A "step" is one pass of the whole hot path (modulate + box sums + combine + divide, plus the fp64
repair of ill-conditioned pixels) over one synthetic input of the workload: one image for cfg0,
cfg1, cfg2 (the headline: the config the north_star target is quoted on), cfg4; 64 frames as 64
back-to-back bf_apply calls on one stream for cfg3 (BASELINE.json configs[3]). Inputs are resident
in HBM before the timed region; L2 is flushed (a 256 MiB write) before every timed step and the
step is timed alone with CUDA events on the launching stream. For N > 1 (torchrun) every rank
filters its own image (independent problems, weak scaling), times are max-reduced over ranks,
value = all ranks' pixels / max time. `e2e` repeats the metric through bf_apply_host (pinned host
input -> device -> host output).

Extra keys: `roofline` (the fused kernel alone against the ALU model),
`hbm_roofline` (the BASELINE metric's HBM fraction), `per_config` (every BASELINE config, each
timed the same way), `parity` (the device fallback / repair counters of one step and the committed
every-pixel full-size result of tests/test_gpu_fullsize.py; the oracle itself runs only in the
cpu_baseline / reference legs), `ncu` (pipe utilisation of the committed capture),
`cpu_baseline` (the oracle on the host cores).
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


def is_u8(spec) -> bool:
    return spec.gen == "ramp" and not spec.as_f32


def frames_per_step(spec) -> int:
    return spec.frames


def config_dict(spec, flush: bool, world: int, n_spatial: int) -> dict:
    return {"workload": f"{spec.name}: {spec.H}x{spec.W} {'uint8' if is_u8(spec) else 'float32'}"
                        f" {spec.gen}, K_s {spec.spatial} sigma_s={spec.sigma_s} r={spec.radius}, "
                        f"K_r {spec.range_kind} sigma_r={spec.sigma_r}, N={spec.n_terms}, D={spec.intensity_max}",
            "H": spec.H, "W": spec.W, "frames_per_step": frames_per_step(spec), "n_spatial": n_spatial,
            "l2": "flushed (256 MiB write) before every timed step" if flush else "not flushed",
            "parallelism": ("single GPU" if world == 1 else
                            f"{world} ranks, the {spec.frames} frames sharded (bf_shard_frames)" if spec.frames > 1
                            else f"dp{world} (independent images per rank)")}


# --------------------------------------------------------------------------------------------
# the CPU oracle (TEST INFRASTRUCTURE used only here, in tests/ and smoke()): the reference arm and
# cpu_baseline. Row bands of a crop are evaluated by os.cpu_count() worker processes
# (tests/fullsize.py: the banded evaluation equals one bf_box call over the crop).
# --------------------------------------------------------------------------------------------

def oracle_rate(spec, side: int, n_spatial: int, pool=None) -> tuple:
    """(MP/s, seconds, description) of the oracle on a side x side crop of the workload."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from fullsize import oracle_banded
    from synth import config_input, config_params
    full = config_input(spec, H=min(spec.H, max(side, 256)), W=min(spec.W, max(side, 256)))
    crop = full[:side, :side].copy()
    params = dict(config_params(spec), n_spatial=n_spatial)
    t0 = time.perf_counter()
    oracle_banded(crop, params, pool=pool)
    dt = time.perf_counter() - t0
    return crop.size / dt / 1e6, dt, (f"{crop.shape[0]}x{crop.shape[1]} crop of the {spec.name} input (frame 0), "
                                      f"oracle.bf.bf_box (fp64 SAT) over {os.cpu_count()} row bands in "
                                      f"{os.cpu_count()} processes")


def cpu_baseline(spec, side: int, n_spatial: int, runs: int = 3) -> dict:
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    n = os.cpu_count() or 1
    with ProcessPoolExecutor(max_workers=n, mp_context=mp.get_context("spawn")) as pool:
        oracle_rate(spec, 128, n_spatial, pool)          # warm the workers (imports)
        res = [oracle_rate(spec, side, n_spatial, pool) for _ in range(runs)]
    rates = [r for r, _, _ in res]
    med = statistics.median(rates)
    return {"value": med, "unit": UNIT, "cores": n, "kind": "oracle", "sample": res[0][2],
            "runs": runs, "statistic": "median", "seconds": [dt for _, dt, _ in res]}


def run_reference(args, spec):
    world, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return 0
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    n = os.cpu_count() or 1
    rates, secs = [], []
    with ProcessPoolExecutor(max_workers=n, mp_context=mp.get_context("spawn")) as pool:
        desc = ""
        for i in range(args.warmup + args.steps):
            r, dt, desc = oracle_rate(spec, args.ref_side, args.n_spatial, pool)
            if i >= args.warmup:
                rates.append(r)
                secs.append(dt)
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(spec, False, 1, args.n_spatial),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": n, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "the fp64 numpy oracle as it stands on the GPU box's host cores (row bands in parallel); "
                    "each step is a bounded crop of the workload"}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------

def committed_json(name: str):
    p = os.path.join(ROOT, "profiles", name)
    return json.load(open(p)) if os.path.exists(p) else None


def rank_frames(pkg, spec, world: int, rank: int) -> range:
    """Frames this rank filters: single-image configs replicate the image on every rank (weak
    scaling); a frame stream (cfg3) is sharded, every frame on exactly one rank (bf_shard_frames,
    strong scaling, no data-path collective)."""
    if spec.frames == 1 or world == 1:
        return range(spec.frames)
    first, count = pkg.shard_frames(spec.frames, world, rank)
    return range(first, first + count)


class Workload:
    """One BASELINE config resident on the device: inputs, outputs, plan, the step callable."""

    def __init__(self, pkg, torch, spec, dev, n_spatial: int, frames: range = None):
        from synth import config_input
        self.spec = spec
        self.plan = pkg.Plan(spatial=spec.spatial, range_kind=spec.range_kind, sigma_s=spec.sigma_s,
                             sigma_r=spec.sigma_r, radius=spec.radius, n_terms=spec.n_terms,
                             intensity_max=spec.intensity_max, n_spatial=n_spatial,
                             input_dtype="u8" if is_u8(spec) else "f32")
        self.frame_ids = frames if frames is not None else range(spec.frames)
        self.nf = len(self.frame_ids)
        self.frames = [config_input(spec, frame=f) for f in self.frame_ids]
        self.inp = torch.from_numpy(self.frames[0] if spec.frames == 1 else __import__("numpy").stack(self.frames)).to(dev)
        self.out = torch.empty(self.inp.shape, dtype=torch.float32, device=dev)
        self.H, self.W = spec.H, spec.W
        self.pkg = pkg
        self.fb = torch.zeros(1, dtype=torch.int64, device=dev)
        self.rep = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = pkg.workspace_size(self.plan, self.H, self.W)
        self.ws = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
        self.wsb = ws

    def args(self, repair=True, counters=False):
        return self.pkg.make_args(workspace=(self.ws.data_ptr(), self.wsb) if self.wsb else (0, 0),
                                  repair_threshold=0.0 if repair else -1.0,
                                  fallback_count=self.fb.data_ptr() if counters else 0,
                                  repaired_count=self.rep.data_ptr() if counters else 0)

    def step(self, stream, args=None):
        """One step: every frame of this rank through bf_apply_ex (cfg3: one call per frame on one
        stream)."""
        n = self.H * self.W
        esz = self.inp.element_size()
        for f in range(self.nf):
            self.pkg.apply_ex(self.plan, self.inp.data_ptr() + f * n * esz, self.out.data_ptr() + f * n * 4, 1,
                              self.H, self.W, stream, args)

    def step_batched(self, stream, args=None):
        self.pkg.apply_ex(self.plan, self.inp.data_ptr(), self.out.data_ptr(), self.nf, self.H, self.W,
                          stream, args)


def timed(torch, stream, fn, steps, warmup, flush, sampler=None):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        for _ in range(steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    return times


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def alu_channels(plan) -> int:
    """C = 4 N_eff box-filtered channels, 4 N_eff - 2 when k = 0 is selected (sin(0 I) == 0)."""
    ks = plan.info()["k"]
    return 4 * len(ks) - (2 if 0 in ks else 0)


def bench_one(pkg, torch, spec, dev, stream, flush, args, steps, warmup, peaks, sampler=None, n_spatial=9,
              frames=None):
    wl = Workload(pkg, torch, spec, dev, n_spatial, frames)
    sptr = stream.cuda_stream
    a = wl.args()
    times = timed(torch, stream, lambda: wl.step(sptr, a), steps, warmup, flush, sampler)
    ms = statistics.median(times) if sampler is None else sum(times) / len(times)
    # the fused kernel alone (no repair launch) for the roofline
    a0 = wl.args(repair=False)
    kt = timed(torch, stream, lambda: wl.step(sptr, a0), max(3, steps // 2), 2, flush)
    kms = statistics.median(kt)
    cfg = pkg.config(wl.plan, spec.H, spec.W)
    px = spec.H * spec.W * wl.nf
    bpp = (1 if is_u8(spec) else 4) + 4
    C = alu_channels(wl.plan)
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 128 * sm_mhz * 1e6
    res = {"ms_per_step": ms, "value": px / 1e6 / (ms / 1e3), "unit": UNIT, "frames_per_step": wl.nf,
           "kernel_ms": kms, "kernel": cfg["kernel"], "launches_per_frame": cfg["launches"] + 1,
           "launch": {"threads_per_cta": cfg["threads_per_cta"], "grid": list(cfg["grid"]), "tile": list(cfg["tile"]),
                      "smem_bytes": cfg["smem_bytes"], "cluster": cfg["cluster"],
                      "terms_per_cta": cfg["terms_per_cta"], "cols_per_thread": cfg["cols_per_thread"]},
           "hbm_frac": px * bpp / (kms / 1e3) / 1e9 / float(peaks["hbm_gbs"]),
           "alu_frac": 8.0 * C * px / (kms / 1e3) / alu_peak, "channels": C}
    if spec.frames > 1:
        bt = timed(torch, stream, lambda: wl.step_batched(sptr, a), steps, warmup, flush)
        res["batched_ms_per_step"] = statistics.median(bt)
        res["batched_value"] = px / 1e6 / (res["batched_ms_per_step"] / 1e3)
        res["per_frame_ms"] = ms / wl.nf
        # the same one-call-per-frame stream captured once into a CUDA graph and replayed
        # (NEXT f4: no per-call host overhead; bf_apply is capturable: no allocation, no sync)
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            wl.step(side.cuda_stream, a)
        stream.wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            wl.step(side.cuda_stream, a)
        gt = timed(torch, stream, g.replay, steps, warmup, flush)
        res["graph_ms_per_step"] = statistics.median(gt)
        res["graph_value"] = px / 1e6 / (res["graph_ms_per_step"] / 1e3)
        del g
    return wl, res, times


def run_ours(args, spec):
    import torch
    from paper_1803_00004_b200 import build
    build.build()
    import paper_1803_00004_b200 as pkg
    from synth import CONFIGS

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    peaks = measured_peaks()

    barrier(world)
    sampler = ClockSampler(local)
    frames = rank_frames(pkg, spec, world, rank)
    sharded = spec.frames > 1 and world > 1
    wl, head, times = bench_one(pkg, torch, spec, dev, stream, flush, args, args.steps, args.warmup, peaks, sampler,
                                args.n_spatial, frames)
    barrier(world)
    total_ms = reduce_max(sum(times), world, dev)
    ms = total_ms / args.steps
    px_step = spec.H * spec.W * wl.nf                               # this rank's pixels per step
    job_px = spec.H * spec.W * (spec.frames if sharded else world * spec.frames)   # all ranks together
    value = job_px * args.steps / 1e6 / (total_ms / 1e3)
    launches = wl.pkg.launches(wl.plan, spec.H, spec.W) + 1      # fused launch(es) + the repair pass

    # parity: device counters of one step, the live sampled check, the committed every-pixel run
    wl.fb.zero_()
    wl.rep.zero_()
    wl.step(stream.cuda_stream, wl.args(counters=True))
    torch.cuda.synchronize()
    parity = {"fallback_pixels": int(wl.fb.item()), "repaired_pixels": int(wl.rep.item())}

    # ---- end to end through the public host API (pinned host buffers, copies inside the timing)
    h_in = [torch.from_numpy(f).pin_memory() for f in wl.frames]
    h_out = torch.empty((spec.H, spec.W), dtype=torch.float32).pin_memory()
    sptr = stream.cuda_stream

    def e2e_step():
        for f in range(wl.nf):
            pkg.apply_host(wl.plan, h_in[f].data_ptr(), h_out.data_ptr(), spec.H, spec.W, sptr)

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier(world)
    e2e_t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_step()
        e2e_t.append(time.perf_counter() - t0)
    e2e_total = reduce_max(sum(e2e_t), world, dev)
    e2e_value = job_px * args.steps / 1e6 / e2e_total

    if rank != 0:
        barrier(world)
        return 0
    committed = committed_json(f"r2_parity_{spec.name}.json")
    if committed:
        parity["full_size_every_pixel"] = {k: committed.get(k) for k in
                                           ("pixels", "max_abs", "rmse", "pass", "cond_min", "n_oracle_fallbacks",
                                            "n_fallback_match", "n_cond_below_1e-3")}
        parity["full_size_every_pixel"]["source"] = f"profiles/r2_parity_{spec.name}.json (tests/test_gpu_fullsize.py)"
    clocks = sampler.summary()
    hbm_peak = float(peaks["hbm_gbs"])
    bpp = (1 if is_u8(spec) else 4) + 4
    alg_bytes = px_step * bpp
    sm_mhz = clocks.get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e12                  # T lane-op/s
    C = alu_channels(wl.plan)
    alu_ops = 8.0 * C * px_step
    kms = head["kernel_ms"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f32 channels, i32 box sums, i64 combine (fp64 repair)", "data": "synthetic",
        "config": config_dict(spec, True, world, args.n_spatial),
        "roofline": {"bound": "alu", "achieved": alu_ops / (kms / 1e3) / 1e12, "peak": alu_peak,
                     "unit": "T lane-op/s", "frac": alu_ops / (kms / 1e3) / 1e12 / alu_peak,
                     "traffic": (committed_json("ncu_traffic.json") or {}).get(spec.name, {}).get("dram_bytes_per_launch"),
                     "kernel": head["kernel"], "kernel_ms": kms, "launch": head["launch"],
                     "algorithmic_ops_per_step": alu_ops, "channels": C,
                     "peak_source": f"148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (B200_PROFILING.md unit counts, "
                                    "SM clock measured under load)",
                     "note": "SURVEY 8(d): >= 8 FP32-lane ops per box-filtered channel-pixel, C = 4 N_eff - 2 "
                             "channels (k = 0 selected: sin(0 I) == 0); the fused kernel timed alone"},
        "hbm_roofline": {"achieved": alg_bytes / (kms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": alg_bytes / (kms / 1e3) / 1e9 / hbm_peak, "algorithmic_bytes_per_step": alg_bytes,
                         "peak_source": peaks["_source"] + " hbm_gbs",
                         "note": "BASELINE metric: image bytes in + out at the measured HBM bandwidth"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(wl.frames[0].nbytes) * wl.nf,
                "d2h_bytes_per_step": int(spec.H * spec.W * 4) * wl.nf},
        "gpu_launches": args.steps * launches * wl.nf,
        "clocks": clocks,
        "parity": parity,
    }
    ncu = committed_json("ncu_pipes.json")
    if ncu and spec.name in ncu:
        line["ncu"] = ncu[spec.name]
    if not args.no_per_config:
        per = {}
        for name in sorted(CONFIGS):
            if name == spec.name:
                per[name] = {k: v for k, v in head.items()}
                continue
            s2 = CONFIGS[name]
            k = 5 if name == "cfg4" else (3 if name == "cfg3" else 10)
            _, r, _ = bench_one(pkg, torch, s2, dev, stream, flush, args, k, 3, peaks, None, args.n_spatial)
            per[name] = r
            torch.cuda.empty_cache()
        line["per_config"] = per
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(spec, args.ref_side, args.n_spatial)
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
    ap.add_argument("--n-spatial", type=int, default=9, help="N_s, the spatial Haar terms (default 9)")
    ap.add_argument("--ref-side", type=int, default=1024, help="side of the oracle's timed crop")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    args = ap.parse_args(argv)
    from synth import CONFIGS
    spec = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, spec)
    return run_ours(args, spec)


if __name__ == "__main__":
    sys.exit(main())
