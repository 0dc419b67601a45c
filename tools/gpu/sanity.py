"""Quick GPU sanity run of every kernel family on small images against the oracle (debug aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_00004_b200 as pkg  # noqa: E402
from oracle import bf, fit  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402


def plan_for(spec, **over):
    p = dict(config_params(spec))
    p.update(over)
    u8 = spec.gen == "ramp" and not spec.as_f32
    return p, pkg.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                       radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                       n_spatial=p.get("n_spatial", 9), input_dtype="u8" if u8 else "f32")


def run(name, cfg, H, W, kernel="auto", **over):
    spec = CONFIGS[cfg]
    p, gp = plan_for(spec, **over)
    img = config_input(spec, H=H, W=W)
    t = torch.from_numpy(img).cuda()
    t0 = time.time()
    out = pkg.bilateral_filter(gp, t, kernel=kernel).cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    dt = time.time() - t0
    ref = bf.bf_box(img, fit.make_plan(**p))
    e = np.abs(out - ref) * 255.0 / spec.intensity_max
    c = pkg.config(gp, H, W, args=pkg.make_args(kernel=kernel))
    print(f"{name:28s} {cfg} {H}x{W} {kernel:8s} max {e.max():.2e} rmse {np.sqrt(np.mean(e*e)):.2e} "
          f"{c['kernel']} G={c['cluster']} cols={c['cols_per_thread']} {dt:.2f}s", flush=True)
    return out


if __name__ == "__main__":
    run("cfg0", "cfg0", 256, 256)
    run("cfg2 small", "cfg2", 333, 361)
    a = run("cfg4 cluster", "cfg4", 419, 430)
    b = run("cfg4 band", "cfg4", 419, 430, kernel="band")
    run("cfg2 wide (G=2)", "cfg2", 333, 361, kernel="ws2wide")
    run("cfg1 N=24 (G=2 cols 1)", "cfg1", 300, 347, n_terms=24)
    run("cfg3 frame", "cfg3", 211, 333)
    print("done")
