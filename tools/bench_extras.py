"""Device timings of the NEXT rows on the B200: CUDA events on the launching
stream, L2 flushed (a 256 MB write) before every repetition, median of 10 after 3 warm-ups.

  f2  Case 1: bf_apply_multi (several range plans over one pass) and the two-phase
      cache (bf_precompute once, bf_apply_cached per range plan) against the full recompute
  f3  richer spatial plans: N_s = 5 (rank 2), 13, 16, 25, 36, 49, 64 (general passes / Form 4)
  f1  the paper-literal z-window (u8)
  --  every kernel on every config it can run (bitwise-equal kernels, A/B)
One line per measurement; `--json PATH` also writes them as a JSON list."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_00004_b200 as pkg  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
RESULTS = []


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def say(name, ms, **kw):
    RESULTS.append(dict(name=name, ms=ms, **kw))
    extra = " ".join(f"{k}={v}" for k, v in kw.items())
    print(f"{name}: {ms:.3f} ms {extra}", flush=True)


def plan_for(spec, **over):
    p = dict(config_params(spec))
    p.update(over)
    u8 = spec.gen == "ramp" and not spec.as_f32
    return pkg.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                    radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                    n_spatial=p.get("n_spatial", 9), haar_levels=p.get("haar_levels", 4),
                    input_dtype="u8" if u8 else "f32", range_window=p.get("range_window", "full"))


def image(cfg):
    im = config_input(CONFIGS[cfg])
    if im.ndim == 3:
        im = im[0]
    return torch.from_numpy(np.ascontiguousarray(im)).cuda()


def case1():
    spec = CONFIGS["cfg2"]
    img = image("cfg2")
    H, W = img.shape
    sigmas = [0.1, 0.05, 0.2, 0.3]
    plans = [plan_for(spec, sigma_r=s) for s in sigmas]
    tukey = plan_for(spec, range_kind="tukey", sigma_r=0.4)
    t1 = timed(lambda: pkg.bilateral_filter(plans[0], img))
    say("f2 cfg2 one plan, full recompute (bf_apply)", t1)
    for n in (2, 3, 4):
        tm = timed(lambda: pkg.bilateral_filter_multi(plans[:n], img))
        say(f"f2 cfg2 {n} sigma_r plans through bf_apply_multi", tm, separate_ms=round(n * t1, 3))
    kmax = max(max(p.info()["k"]) for p in plans + [tukey]) + 1
    out = torch.empty((H, W), dtype=torch.float32, device="cuda")
    tp = timed(lambda: pkg.RangeCache(plans[0], img, kmax))
    cache = pkg.RangeCache(plans[0], img, kmax)
    say(f"f2 cfg2 bf_precompute k < {kmax}", tp, cache_bytes=int(cache.buf.numel()))
    for p, name in zip(plans + [tukey], [f"gaussian sigma_r={s}" for s in sigmas] + ["tukey 0.4"]):
        tc = timed(lambda p=p: cache.apply(p, out))
        ref = pkg.bilateral_filter(p, img)
        same = bool(torch.equal(ref, cache.apply(p, out)))
        say(f"f2 cfg2 bf_apply_cached {name}", tc, bitwise_equal_to_bf_apply=same,
            n_terms=len(p.info()["k"]))


def spatial():
    for cfg in ("cfg0", "cfg1", "cfg2"):
        sp = CONFIGS[cfg]
        im = image(cfg)
        for ns in (9, 5, 13, 16, 25, 36, 49, 64):
            try:
                p = plan_for(sp, n_spatial=ns)
                inf = p.info()
                t = timed(lambda: pkg.bilateral_filter(p, im))
            except Exception as e:  # noqa: BLE001
                print(f"f3 {cfg} N_s={ns}: {e}")
                continue
            say(f"f3 {cfg} N_s={ns}", t, rank=inf["spatial_rank"], passes=inf["spatial_passes"],
                mp_s=round(im.numel() / t / 1e3))


def literal():
    for cfg in ("cfg0", "cfg3"):
        sp = CONFIGS[cfg]
        im = image(cfg)
        p = plan_for(sp)
        pl = plan_for(sp, range_window="literal")
        t0 = timed(lambda: pkg.bilateral_filter(p, im))
        tl = timed(lambda: pkg.bilateral_filter(pl, im))
        say(f"f1 {cfg} literal window T_r={pl.info()['T_range']:.1f}", tl, mp_s=round(im.numel() / tl / 1e3),
            t_eq_d_ms=round(t0, 4))


def kernels():
    for cfg in ("cfg0", "cfg1", "cfg2", "cfg3", "cfg4"):
        sp = CONFIGS[cfg]
        im = image(cfg)
        p = plan_for(sp)
        ref = None
        for k in ("ws2", "ws2wide", "ws", "band"):
            if cfg == "cfg4" and k in ("ws", "band"):
                continue   # (the barrier-interval kernel needs several passes at r = 192: tens of ms)
            try:
                o = pkg.bilateral_filter(p, im, kernel=k, repair_threshold=-1.0)
                t = timed(lambda: pkg.bilateral_filter(p, im, kernel=k, repair_threshold=-1.0),
                          reps=5 if cfg == "cfg4" else 10)
            except Exception as e:  # noqa: BLE001
                print(f"kernel {cfg} {k}: {e}")
                continue
            same = None if ref is None else bool(torch.equal(ref, o))
            ref = o if ref is None else ref
            say(f"kernel {cfg} {k}", t, bitwise_equal_to_first=same)


def main():
    which = sys.argv[1].split(",") if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else \
        ["case1", "spatial", "literal", "kernels"]
    for w in which:
        globals()[w]()
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(RESULTS, f, indent=1)


if __name__ == "__main__":
    main()
