"""Every-pixel parity at the BASELINE configs' FULL sizes (north_star target; SURVEY 8(d) "check
every pixel of every config"): the CUDA path, launched exactly as bench.py launches it, against
the oracle evaluated on every pixel by the tiled multi-process harness of tests/fullsize.py.
cfg3 runs all 64 frames as 64 back-to-back bf_apply calls on one stream (BASELINE configs[3]).

Tolerance (north_star): max-abs <= 1e-3 and RMSE <= 1e-4 on the [0, 255] scale, on every pixel,
including the ill-conditioned ones (small den / sum K~_s) and the oracle's fallback pixels
(den <= 0, reading Q18), where the GPU must take the same decision.

Set BF_PARITY_OUT=<dir> to write one JSON summary per config (worst pixels, conditioning,
fallbacks) there; tools/parity_fullsize.py does the same outside pytest."""
import json
import os

import numpy as np
import pytest

from synth import CONFIGS, config_input, config_params

from fullsize import oracle_banded, oracle_frames, summarise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    from paper_1803_00004_b200 import build
    build.build()
    import paper_1803_00004_b200 as pkg
    assert torch.cuda.is_available()
    return pkg, torch


def gpu_plan(pkg, spec):
    u8 = spec.gen == "ramp" and not spec.as_f32
    p = config_params(spec)
    return pkg.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                    radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                    input_dtype="u8" if u8 else "f32")


def record(name, summ):
    d = os.environ.get("BF_PARITY_OUT")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"parity_{name}.json"), "w") as f:
            json.dump(summ, f, indent=1)
    w = summ["worst"][0] if summ.get("worst") else {}
    print(f"\n[parity {name}] max-abs {summ['max_abs']:.3e} rmse {summ['rmse']:.3e} cond_min {summ['cond_min']:.2e} "
          f"oracle fallbacks {summ['n_oracle_fallbacks']} matched {summ['n_fallback_match']} worst {w}")


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg4"])
def test_full_size_every_pixel(gpu, cfg):
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec)
    plan = gpu_plan(pkg, spec)
    t = torch.from_numpy(img).cuda()
    got = pkg.bilateral_filter(plan, t).cpu().numpy()
    torch.cuda.synchronize()
    del t
    ref, cond, fb = oracle_banded(img, config_params(spec))
    summ = summarise(got, ref, cond, fb, spec.intensity_max, img)
    summ["config"] = cfg
    record(cfg, summ)
    assert summ["finite"]
    assert summ["n_fallback_match"] == summ["n_oracle_fallbacks"], summ["oracle_fallbacks"]
    assert summ["pass"], (summ["max_abs"], summ["rmse"], summ["worst"][:3])


def test_cfg3_all_64_frames_every_pixel(gpu):
    pkg, torch = gpu
    spec = CONFIGS["cfg3"]
    frames = [config_input(spec, frame=f) for f in range(spec.frames)]
    plan = gpu_plan(pkg, spec)
    dev_in = [torch.from_numpy(f).cuda() for f in frames]
    dev_out = [torch.empty(f.shape, dtype=torch.float32, device="cuda") for f in frames]
    s = torch.cuda.current_stream().cuda_stream
    H, W = frames[0].shape
    for i, o in zip(dev_in, dev_out):          # 64 back-to-back calls on one stream
        pkg.apply(plan, i.data_ptr(), o.data_ptr(), H, W, s)
    torch.cuda.synchronize()
    got = [o.cpu().numpy() for o in dev_out]
    refs = oracle_frames(frames, config_params(spec))
    per = []
    for f, (g, (ref, cond, fb)) in enumerate(zip(got, refs)):
        sm = summarise(g, ref, cond, fb, 255.0, frames[f], n_worst=3)
        sm["frame"] = f
        per.append(sm)
    summ = {"config": "cfg3", "frames": len(per), "pixels": int(sum(p["pixels"] for p in per)),
            "max_abs": max(p["max_abs"] for p in per),
            "rmse": float(np.sqrt(np.mean([p["rmse"] ** 2 for p in per]))),
            "finite": all(p["finite"] for p in per),
            "cond_min": min(p["cond_min"] for p in per),
            "n_oracle_fallbacks": sum(p["n_oracle_fallbacks"] for p in per),
            "n_fallback_match": sum(p["n_fallback_match"] for p in per),
            "fallback_frames": {p["frame"]: p["oracle_fallbacks"] for p in per if p["n_oracle_fallbacks"]},
            "worst": sorted((dict(w, frame=p["frame"]) for p in per for w in p["worst"]), key=lambda w: -w["err"])[:8],
            "worst_conditioned": sorted((dict(w, frame=p["frame"]) for p in per for w in p["worst_conditioned"]),
                                        key=lambda w: w["cond"])[:8],
            "per_frame_max_abs": [p["max_abs"] for p in per]}
    summ["pass"] = bool(summ["finite"] and summ["max_abs"] <= 1e-3 and summ["rmse"] <= 1e-4)
    record("cfg3", summ)
    assert summ["finite"]
    assert summ["n_fallback_match"] == summ["n_oracle_fallbacks"], summ["fallback_frames"]
    assert summ["pass"], (summ["max_abs"], summ["rmse"], summ["worst"][:3])
