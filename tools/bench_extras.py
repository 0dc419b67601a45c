"""Device timings of the NEXT rows on the B200 (CUDA events, L2 flushed, median of 10 after 3
warm-ups): Case 1 multi-plan sharing (bf_apply_multi, f2), rank-2 three-box plans (N_s = 5, f3),
and both kernels per config. Prints one line per measurement."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_00004_b200 as pkg  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


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


def plan_for(spec, **over):
    p = dict(config_params(spec))
    p.update(over)
    u8 = spec.gen == "ramp" and not spec.as_f32
    return pkg.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                    radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                    n_spatial=p.get("n_spatial", 9), input_dtype="u8" if u8 else "f32")


def main():
    spec = CONFIGS["cfg2"]
    img = torch.from_numpy(config_input(spec)).cuda()
    H, W = img.shape
    sigmas = [0.1, 0.05, 0.2, 0.3]
    plans = [plan_for(spec, sigma_r=s) for s in sigmas]
    t1 = timed(lambda: pkg.bilateral_filter(plans[0], img))
    print(f"cfg2 single plan: {t1:.3f} ms")
    for n in (2, 3, 4):
        tm = timed(lambda: pkg.bilateral_filter_multi(plans[:n], img))
        ts = sum(timed(lambda p=p: pkg.bilateral_filter(p, img)) for p in plans[:n])
        print(f"cfg2 {n} sigma_r plans: multi {tm:.3f} ms vs {n} separate {ts:.3f} ms ({ts / tm:.2f}x)")
    for cfg in ("cfg0", "cfg1", "cfg2"):
        sp = CONFIGS[cfg]
        im = torch.from_numpy(config_input(sp)).cuda()
        for ns in (9, 5):
            p = plan_for(sp, n_spatial=ns)
            t = timed(lambda: pkg.bilateral_filter(p, im))
            print(f"{cfg} N_s={ns} (rank {p.info()['spatial_rank']}): {t:.3f} ms, "
                  f"{im.numel() / t / 1e3:.0f} MP/s")
    for cfg in ("cfg0", "cfg3"):   # the paper-literal window (NEXT f1), u8 configs
        sp = CONFIGS[cfg]
        im = torch.from_numpy(config_input(sp)).cuda()
        p = plan_for(sp)
        prm = config_params(sp)
        pl = pkg.Plan(spatial=prm["spatial"], range_kind=prm["range_kind"], sigma_s=prm["sigma_s"],
                      sigma_r=prm["sigma_r"], radius=prm["radius"], n_terms=prm["n_terms"], input_dtype="u8",
                      range_window="literal")
        t0 = timed(lambda: pkg.bilateral_filter(p, im))
        tl = timed(lambda: pkg.bilateral_filter(pl, im))
        print(f"{cfg} literal window T_r={pl.info()['T_range']:.1f}: {tl:.3f} ms ({im.numel() / tl / 1e3:.0f} MP/s) "
              f"vs T=D hot path {t0:.3f} ms")
    for cfg in ("cfg0", "cfg1", "cfg2", "cfg3"):
        sp = CONFIGS[cfg]
        im = torch.from_numpy(config_input(sp)).cuda()
        p = plan_for(sp)
        for k in ("band", "ws", "ws2"):
            os.environ["BF_KERNEL"] = k
            t = timed(lambda: pkg.bilateral_filter(p, im))
            print(f"{cfg} kernel={k}: {t:.3f} ms")
        os.environ.pop("BF_KERNEL")


if __name__ == "__main__":
    main()
