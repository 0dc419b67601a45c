"""GPU tests of the boundary's contract and of the newer paths: CUDA-graph capture (no allocation,
no synchronisation inside bf_apply), the fallback counter / mask ("the pixel is counted"),
the Case 1 cache and the Case 2 LUT, the cluster-split kernel, the
fp64 repair of ill-conditioned pixels (reading Q27) and row ranges. Parity tolerance as in
test_gpu_parity.py (north_star: max-abs <= 1e-3, RMSE <= 1e-4 on the [0, 255] scale)."""
import math

import numpy as np
import pytest

from oracle import bf, fit
from synth import CONFIGS, config_input, config_params

pytestmark = pytest.mark.gpu

MAX_ABS = 1e-3
RMSE = 1e-4


@pytest.fixture(scope="module")
def gpu():
    import torch
    from paper_1803_00004_b200 import build
    build.build()
    import paper_1803_00004_b200 as pkg
    assert torch.cuda.is_available()
    return pkg, torch


def plans(pkg, spec, **over):
    p = dict(config_params(spec))
    p.update(over)
    u8 = spec.gen == "ramp" and not spec.as_f32
    gp = pkg.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                  radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                  n_spatial=p.get("n_spatial", 9), input_dtype="u8" if u8 else "f32")
    return gp, fit.make_plan(**p)


def parity(got, ref, D, what=""):
    e = np.abs(np.asarray(got, np.float64) - ref) * (255.0 / D)
    mx, rm = float(e.max()), float(np.sqrt(np.mean(e * e)))
    assert np.all(np.isfinite(got)), what
    assert mx <= MAX_ABS and rm <= RMSE, f"{what}: max-abs {mx:.3e} rmse {rm:.3e}"


def gpu_out(pkg, torch, plan, img, **kw):
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    o = pkg.bilateral_filter(plan, t, **kw)
    torch.cuda.synchronize()
    return o.cpu().numpy()


@pytest.mark.parametrize("cfg,H,W,kernel", [("cfg0", 256, 256, "auto"), ("cfg2", 300, 420, "auto"),
                                            ("cfg4", 420, 400, "auto"), ("cfg4", 300, 260, "band"),
                                            ("cfg3", 200, 333, "auto")])
def test_graph_capture_matches_eager(gpu, cfg, H, W, kernel):
    """bf_apply (and the workspace passes of a forced kernel 1, the repair pass, the cluster launch)
    captured into a CUDA graph and replayed equals the eager call bitwise: nothing inside
    allocates or synchronises."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    gp, _ = plans(pkg, spec)
    img = torch.from_numpy(config_input(spec, H=H, W=W)).cuda()
    eager = pkg.bilateral_filter(gp, img, kernel=kernel).clone()
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        pkg.bilateral_filter(gp, img, out=out, kernel=kernel)     # warm-up on the side stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    out.fill_(float("nan"))
    with torch.cuda.graph(g):
        pkg.bilateral_filter(gp, img, out=out, kernel=kernel)
    out.fill_(float("nan"))
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


def test_fallback_counter_and_mask_cfg3_frame12(gpu):
    """cfg3 frame 12 at full size: the oracle has pixels with den <= 0 (out = I(x), Q18); the
    library counts exactly those (device counter) and marks them (device mask), and their outputs
    equal I(x)."""
    pkg, torch = gpu
    spec = CONFIGS["cfg3"]
    img = config_input(spec, frame=12)
    gp, op = plans(pkg, spec)
    ref, num, den, fb = bf.bf_box(img, op, return_parts=True)
    assert fb.sum() >= 1
    t = torch.from_numpy(img).cuda()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    mask = torch.full(img.shape, 7, dtype=torch.uint8, device="cuda")
    out = pkg.bilateral_filter(gp, t, fallback_count=cnt, fallback_mask=mask).cpu().numpy()
    m = mask.cpu().numpy()
    assert set(np.unique(m)) <= {0, 1}
    assert int(cnt.item()) == int(fb.sum())
    assert np.array_equal(m.astype(bool), fb)
    assert np.array_equal(out[fb], img[fb].astype(np.float32))
    parity(out, ref, 255.0, "cfg3 frame 12")


@pytest.mark.parametrize("cfg,H,W,variants", [
    ("cfg2", 300, 420, [dict(sigma_r=0.05), dict(sigma_r=0.1), dict(sigma_r=0.2),
                        dict(range_kind="tukey", sigma_r=0.16, n_terms=12)]),
    ("cfg0", 256, 256, [dict(sigma_r=15.0), dict(sigma_r=30.0, n_terms=16), dict(range_kind="tukey", sigma_r=40.0)]),
])
def test_case1_cache_matches_apply_and_oracle(gpu, cfg, H, W, variants):
    """Case 1: the box-filtered channels of k < k_count computed once
    (bf_precompute); each range plan chosen afterwards is a combine-only pass (bf_apply_cached)
    whose output matches the oracle within the tolerance, and bf_apply to the rounding of the
    cached F = round(sum_b ax_b H_b / 2^32) (bf_apply keeps the per-box sums exact)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    base, _ = plans(pkg, spec)
    t = torch.from_numpy(img).cuda()
    cache = pkg.RangeCache(base, t, k_count=32)
    for v in variants:
        gp, op = plans(pkg, spec, **v)
        assert max(gp.info()["k"]) < 32
        got = cache.apply(gp).cpu().numpy()
        want = pkg.bilateral_filter(gp, t).cpu().numpy()
        e = np.abs(got.astype(np.float64) - want) * (255.0 / spec.intensity_max)
        assert float(e.max()) <= 1e-4 and float(np.sqrt(np.mean(e * e))) <= 1e-5, (v, float(e.max()))
        parity(got, bf.bf_box(img, op), spec.intensity_max, f"{cfg} {v}")
    other, _ = plans(pkg, spec, sigma_s=2.0, radius=6)
    with pytest.raises(pkg.BFError):
        cache.apply(other)                       # another spatial plan: refused


@pytest.mark.parametrize("cfg,H,W", [("cfg0", 256, 256), ("cfg3", 200, 333)])
def test_case2_lut_equals_direct_trig(gpu, cfg, H, W):
    """Case 2: the u8 path's 256-entry (cos, sin) table gives bitwise the output of
    evaluating the trig functions per tap."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, _ = plans(pkg, spec)
    lut = gpu_out(pkg, torch, gp, img, kernel="band")
    direct = gpu_out(pkg, torch, gp, img, kernel="band", u8_trig="direct")
    assert np.array_equal(lut, direct)
    # the default kernel (2b: per-box sums, no rounded F) agrees to F's rounding
    e = np.abs(lut.astype(np.float64) - gpu_out(pkg, torch, gp, img))
    assert float(e.max()) <= 1e-4 and float(np.sqrt(np.mean(e * e))) <= 1e-5


@pytest.mark.parametrize("cfg,H,W,over,want", [
    ("cfg1", 300, 347, {"n_terms": 24}, (1, 2)),                    # r = 24: one column, 2 CTAs x 16 terms
    ("cfg1", 257, 300, {"n_terms": 32, "sigma_r": 8.0}, (1, 2)),
    ("cfg4", 419, 430, {}, (2, 3)),                                 # r = 192: two columns, 3 CTAs x 8 terms
    ("cfg4", 400, 500, {"range_kind": "gaussian", "sigma_r": 12.0, "n_terms": 32}, (2, 4)),
    ("cfg4", 350, 610, {"n_terms": 8}, (2, 1)),                     # one CTA, two columns
    ("cfg2", 333, 361, {"n_terms": 24}, (1, 2)),
])
def test_cluster_split_kernel(gpu, cfg, H, W, over, want):
    """The range terms split over a CTA cluster (num / den partials reduced through distributed
    shared memory) and two columns per vertical-pass thread: parity with the oracle, one launch,
    and bitwise independence of the band height (every band restarts its exact sliding sums)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, op = plans(pkg, spec, **over)
    c = pkg.config(gp, H, W)
    assert (c["cols_per_thread"], c["cluster"], c["launches"]) == want + (1,), c
    a = gpu_out(pkg, torch, gp, img)
    parity(a, bf.bf_box(img, op), spec.intensity_max, f"{cfg} {over}")
    assert np.array_equal(a, gpu_out(pkg, torch, gp, img, band_rows=16))


def test_two_columns_forced_on_cfg2(gpu):
    pkg, torch = gpu
    spec = CONFIGS["cfg2"]
    img = config_input(spec, H=333, W=761)
    gp, op = plans(pkg, spec)
    c = pkg.config(gp, 333, 761, args=pkg.make_args(kernel="ws2wide"))
    assert (c["cols_per_thread"], c["cluster"]) == (2, 2)
    parity(gpu_out(pkg, torch, gp, img, kernel="ws2wide"), bf.bf_box(img, op), 1.0, "cfg2 ws2wide")


@pytest.mark.parametrize("cfg,H,W,over", [("cfg2", 150, 210, {}), ("cfg0", 160, 200, {}),
                                          ("cfg1", 150, 210, {"n_spatial": 5}), ("cfg4", 170, 190, {})])
def test_repair_pass_alone_reproduces_oracle(gpu, cfg, H, W, over):
    """With the repair threshold above every pixel's conditioning, every pixel is re-evaluated by
    the fp64 repair pass (the direct double loop of pin P1): the output then equals the oracle's
    to float32 rounding, including its fallback pixels. (Images of <= 32768 pixels: the repair
    list's capacity per call.)"""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, op = plans(pkg, spec, **over)
    ref = bf.bf_box(img, op)
    got = gpu_out(pkg, torch, gp, img, repair_threshold=1e30).astype(np.float64)
    tol = 4 * np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64) + 1e-9 * spec.intensity_max
    assert np.all(np.abs(got - ref) <= tol), float(np.max(np.abs(got - ref) / tol))
    off = gpu_out(pkg, torch, gp, img, repair_threshold=-1).astype(np.float64)
    assert np.all(np.isfinite(off))


def test_row_range(gpu):
    """bf_apply_ex over output rows [a, b) writes exactly those rows, equal to the full call's."""
    pkg, torch = gpu
    spec = CONFIGS["cfg2"]
    img = config_input(spec, H=400, W=300)
    gp, _ = plans(pkg, spec)
    t = torch.from_numpy(img).cuda()
    full = pkg.bilateral_filter(gp, t)
    part = torch.full_like(full, float("nan"))
    s = torch.cuda.current_stream().cuda_stream
    pkg.apply_ex(gp, t.data_ptr(), part.data_ptr(), 1, 400, 300, s, pkg.make_args(rows=(123, 311)))
    torch.cuda.synchronize()
    f, p = full.cpu().numpy(), part.cpu().numpy()
    assert np.array_equal(p[123:311], f[123:311])
    assert np.all(np.isnan(p[:123])) and np.all(np.isnan(p[311:]))


def test_graph_captured_frame_stream(gpu):
    """NEXT f4 (BASELINE configs[3], "one bf_apply per frame on one stream"): a stream of per-frame
    bf_apply calls captured once into a CUDA graph (each call claims its own repair slot at capture
    time; on one stream the calls stay ordered) and replayed gives every frame bitwise as the eager
    calls, which equal bf_apply_batched's frames."""
    pkg, torch = gpu
    spec = CONFIGS["cfg3"]
    H, W, F = 120, 200, 20                       # more frames than repair slots (16)
    frames = torch.from_numpy(np.stack([config_input(spec, H=H, W=W, frame=f) for f in range(F)])).cuda()
    gp, _ = plans(pkg, spec)
    eager = torch.stack([pkg.bilateral_filter(gp, frames[f]) for f in range(F)])
    batched = pkg.bilateral_filter(gp, frames)
    assert torch.equal(eager, batched)
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in range(F):
            pkg.bilateral_filter(gp, frames[f], out=out[f], stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for f in range(F):
            pkg.bilateral_filter(gp, frames[f], out=out[f], stream=s)
    out.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
