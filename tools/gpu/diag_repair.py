"""Diagnostic (not a test): how many pixels the fp64 repair pass re-evaluates per config at several
thresholds tau (den / sum K~_s < tau), and what the call costs with and without it.

    python tools/gpu/diag_repair.py [cfg ...]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1803_00004_b200 as pkg  # noqa: E402
from synth import CONFIGS, config_input  # noqa: E402


def main():
    cfgs = sys.argv[1:] or ["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for c in cfgs:
        spec = CONFIGS[c]
        u8 = spec.gen == "ramp" and not spec.as_f32
        plan = pkg.Plan(spatial=spec.spatial, range_kind=spec.range_kind, sigma_s=spec.sigma_s, sigma_r=spec.sigma_r,
                        radius=spec.radius, n_terms=spec.n_terms, intensity_max=spec.intensity_max,
                        input_dtype="u8" if u8 else "f32")
        nf = min(spec.frames, 8)
        x = torch.from_numpy(__import__("numpy").stack([config_input(spec, frame=f) for f in range(nf)])).cuda()
        y = torch.empty(x.shape, dtype=torch.float32, device="cuda")
        for tau in (-1.0, 0.0, 0.015, 0.008, 0.004, 0.002):
            rep = torch.zeros(1, dtype=torch.int64, device="cuda")
            ts = []
            for i in range(4):
                rep.zero_()
                flush.zero_()
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for f in range(nf):
                    pkg.bilateral_filter(plan, x[f], out=y[f], repair_threshold=tau, repaired_count=rep)
                e.record()
                e.synchronize()
                if i:
                    ts.append(a.elapsed_time(e) / nf)
            print(f"{c} tau {tau:7.4f}: repaired {int(rep.item()) / nf:10.1f} px/frame  {statistics.median(ts):8.3f} ms/frame",
                  flush=True)


if __name__ == "__main__":
    main()
