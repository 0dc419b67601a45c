"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs. Tolerance (BASELINE.json north_star): max-abs <= 1e-3 and RMSE <= 1e-4 on intensities
scaled to [0, 255]. Full images at sizes the oracle finishes in seconds (several strips/bands
and ragged tails), sampled pixels at the configs' full sizes, and edge cases."""
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


def make_plans(pkg, params, dtype, **over):
    p = dict(params)
    p.update(over)
    gp = pkg.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                  radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                  n_spatial=p.get("n_spatial", 9), input_dtype="u8" if dtype == np.uint8 else "f32")
    op = fit.make_plan(**p)
    return gp, op


def run_gpu(pkg, torch, plan, img, **kw):
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    out = pkg.bilateral_filter(plan, t, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def assert_parity(got, ref, D, what=""):
    e = np.abs(got - ref) * (255.0 / D)
    mx, rm = float(e.max()), float(np.sqrt(np.mean(e * e)))
    assert np.all(np.isfinite(got)), what
    assert mx <= MAX_ABS and rm <= RMSE, f"{what}: max-abs {mx:.3e} rmse {rm:.3e}"
    return mx, rm


def assert_close(a, b, D, what=""):
    """Two GPU paths that differ only in the rounding of the horizontally weighted box sums F
    (kernels 1/2 round F to an integer, kernel 2b keeps the per-box sums exact): far below the
    tolerance (max-abs 1e-4, RMSE 1e-5 on the [0, 255] scale; the repair pass covers the
    ill-conditioned pixels in both)."""
    e = np.abs(a - b) * (255.0 / D)
    assert float(e.max()) <= 1e-4 and float(np.sqrt(np.mean(e * e))) <= 1e-5, (what, float(e.max()))


# ------------------------------------------------------------------ whole images vs the oracle

SMALL = {
    "cfg0": (256, 256),          # cfg0 at its full size
    "cfg1": (300, 347),
    "cfg2": (333, 361),          # r = 48: 3 strips (TW = 160) + ragged tail, 2 bands
    "cfg3": (211, 333),
    "cfg4": (419, 430),          # r = 192, Tukey, 24 terms: 2 passes, 4 strips
}


@pytest.mark.parametrize("cfg", sorted(SMALL))
def test_config_small_full_image(gpu, cfg):
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    H, W = SMALL[cfg]
    img = config_input(spec, H=H, W=W)
    gp, op = make_plans(pkg, config_params(spec), img.dtype)
    got = run_gpu(pkg, torch, gp, img)
    ref = bf.bf_box(img, op)
    assert_parity(got, ref, spec.intensity_max, cfg)


def sample_pixels(H, W, r, n, seed):
    rng = np.random.default_rng(seed)
    pts = {(0, 0), (0, W - 1), (H - 1, 0), (H - 1, W - 1), (H // 2, W // 2), (min(r, H - 1), min(r, W - 1)),
           (H - 1 - min(r, H - 1), W // 3)}
    while len(pts) < n:
        pts.add((int(rng.integers(0, H)), int(rng.integers(0, W))))
    return sorted(pts)


@pytest.mark.parametrize("cfg,n", [("cfg1", 48), ("cfg2", 48), ("cfg3", 32), ("cfg4", 24)])
def test_config_full_size_sampled(gpu, cfg, n):
    """Full BASELINE size, launched exactly as bench.py launches it; the oracle evaluates the
    same approximation directly at sampled pixels (pin P1 ties it to the box evaluation)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec)
    gp, op = make_plans(pkg, config_params(spec), img.dtype)
    got = run_gpu(pkg, torch, gp, img)
    pts = sample_pixels(spec.H, spec.W, spec.radius, n, seed=7)
    ref, _, _ = bf.bf_direct(img, op, pixels=pts)
    vals = np.array([got[y, x] for (y, x) in pts])
    assert_parity(vals, ref, spec.intensity_max, cfg)
    # properties that hold at any size: finite, within [0, D] up to the approximation slack
    assert np.all(np.isfinite(got))
    D = spec.intensity_max
    assert got.min() > -0.1 * D and got.max() < 1.1 * D


def test_cfg3_batched_frames_match_single_calls(gpu):
    pkg, torch = gpu
    spec = CONFIGS["cfg3"]
    H, W = 120, 207
    frames = np.stack([config_input(spec, frame=f, H=H, W=W) for f in range(3)])
    gp, op = make_plans(pkg, config_params(spec), frames.dtype)
    t = torch.from_numpy(frames).cuda()
    outb = pkg.bilateral_filter(gp, t).cpu().numpy()
    for f in range(3):
        single = run_gpu(pkg, torch, gp, frames[f])
        assert np.array_equal(outb[f], single.astype(np.float32))
        assert_parity(single, bf.bf_box(frames[f], op), 255.0, f"frame {f}")


@pytest.mark.parametrize("cfg,H,W", [("cfg2", 2048, 600), ("cfg4", 2100, 520), ("cfg0", 1100, 1000), ("cfg1", 90, 77)])
def test_host_path_matches_device_path(gpu, cfg, H, W):
    """bf_apply_host pipelines row chunks (input piece j+1 copied while chunk j is filtered and
    chunk j-1 copied back; each chunk a separate row-range launch with its own band tiling). The
    integer pipeline makes every output independent of the tiling, so the host path must equal
    the one-launch device path bitwise (cfg4: two passes through the workspace per chunk)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, _ = make_plans(pkg, config_params(spec), img.dtype)
    dev = run_gpu(pkg, torch, gp, img)
    h_in = torch.from_numpy(img).pin_memory()
    h_out = torch.full((H, W), float("nan"), dtype=torch.float32).pin_memory()
    pkg.apply_host(gp, h_in.data_ptr(), h_out.data_ptr(), H, W, torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(h_out.numpy().astype(np.float64), dev)


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("H,W", [(1, 1), (1, 57), (61, 1), (5, 7), (7, 300), (300, 6), (17, 33)])
def test_degenerate_shapes(gpu, H, W):
    pkg, torch = gpu
    spec = CONFIGS["cfg1"]
    img = config_input(spec, H=max(H, 2), W=max(W, 2))[:H, :W].copy()
    gp, op = make_plans(pkg, config_params(spec), img.dtype)
    assert_parity(run_gpu(pkg, torch, gp, img), bf.bf_box(img, op), 255.0, f"{H}x{W}")


@pytest.mark.parametrize("cfg,W", [("cfg0", 40), ("cfg0", 100), ("cfg0", 170), ("cfg3", 230), ("cfg1", 75),
                                   ("cfg1", 140), ("cfg1", 290), ("cfg2", 150)])
def test_strip_widths_and_warp_role_maps(gpu, cfg, W):
    """Strips that leave different numbers of FH / V warps working (kernel 2b's warp-role map,
    the per-sub-partition deal of the band's initial state and the TMEM blocks all depend on
    them): whole image against the oracle, and the map a permutation of the 24 warps."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    H = 70
    img = config_input(spec, H=H, W=W)
    gp, op = make_plans(pkg, config_params(spec), img.dtype)
    c = pkg.config(gp, H, W)
    assert c["kernel"] == "bf_ws2_kernel" and sorted(c["warp_map"]) == list(range(24)), c
    assert_parity(run_gpu(pkg, torch, gp, img), bf.bf_box(img, op), spec.intensity_max, f"{cfg} W={W}")


def test_constant_image(gpu):
    pkg, torch = gpu
    img = np.full((70, 90), 0.625, dtype=np.float32)
    gp, op = make_plans(pkg, config_params(CONFIGS["cfg2"]), img.dtype, radius=20, sigma_s=6.0)
    got = run_gpu(pkg, torch, gp, img)
    assert np.max(np.abs(got - 0.625)) * 255 <= MAX_ABS


def test_radius_zero_identity(gpu):
    pkg, torch = gpu
    img = config_input(CONFIGS["cfg0"], H=40, W=50)
    gp, op = make_plans(pkg, config_params(CONFIGS["cfg0"]), img.dtype, radius=0)
    assert_parity(run_gpu(pkg, torch, gp, img), img.astype(np.float64), 255.0, "r=0")


def test_infinite_sigma_r(gpu):
    pkg, torch = gpu
    img = config_input(CONFIGS["cfg1"], H=64, W=80)
    gp, op = make_plans(pkg, config_params(CONFIGS["cfg1"]), img.dtype, sigma_r=math.inf)
    assert gp.info()["k"] == [0]
    assert_parity(run_gpu(pkg, torch, gp, img), bf.bf_box(img, op), 255.0, "sigma_r=inf")


def test_u8_and_f32_inputs_agree(gpu):
    pkg, torch = gpu
    spec = CONFIGS["cfg0"]
    img8 = config_input(spec, H=90, W=110)
    g8, op = make_plans(pkg, config_params(spec), np.uint8)
    g32, _ = make_plans(pkg, config_params(spec), np.float32)
    o8 = run_gpu(pkg, torch, g8, img8)
    o32 = run_gpu(pkg, torch, g32, img8.astype(np.float32))
    ref = bf.bf_box(img8, op)
    assert_parity(o8, ref, 255.0, "u8")
    assert_parity(o32, ref, 255.0, "f32")


def test_deterministic(gpu):
    pkg, torch = gpu
    spec = CONFIGS["cfg2"]
    img = config_input(spec, H=200, W=230)
    gp, _ = make_plans(pkg, config_params(spec), img.dtype)
    a = run_gpu(pkg, torch, gp, img)
    b = run_gpu(pkg, torch, gp, img)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg,H,W", [("cfg0", 150, 230), ("cfg1", 170, 260), ("cfg2", 140, 250)])
def test_rank2_three_box_plan(gpu, cfg, H, W):
    """N_s = 5 (f1 + f2 + f3, the paper's three boxes): a rank-2 spatial kernel, run as two
    box-pair terms (NEXT f3). Both kernels, against the oracle's box evaluation of the same plan."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, op = make_plans(pkg, config_params(spec), img.dtype, n_spatial=5)
    assert gp.info()["spatial_rank"] == 2 and not gp.info()["separable"]
    ref, _, den, _ = bf.bf_box(img, op, return_parts=True)
    # this kernel has negative corners: den can approach 0 (cfg1 has 4 pixels with den <= 0), where
    # out = num / den amplifies the integer path's rounding by sum(K~_s) / |den| and the fallback
    # decision (den <= 0, Q18) rides on it. With the fp64 repair pass (reading Q27) every pixel is
    # held to the tolerance, the oracle's fallback pixels included (Q26).
    cond = den / fit.spatial_kernel_values(op.sp).sum()
    outs = []
    for k in ("band", "ws"):
        got = run_gpu(pkg, torch, gp, img, kernel=k)
        assert np.all(np.isfinite(got))
        assert_parity(got, ref, spec.intensity_max, f"{cfg} N_s=5 {k} (every pixel, cond_min {cond.min():.1e})")
        fb = ~(den > 0)
        assert np.array_equal(got[fb], img[fb].astype(np.float32)), "fallback pixels: out = I(x)"
        # the fused path alone (repair off) agrees between the two kernels bitwise
        outs.append(run_gpu(pkg, torch, gp, img, kernel=k, repair_threshold=-1))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("cfg,H,W", [("cfg0", 256, 256), ("cfg1", 150, 347), ("cfg2", 333, 361), ("cfg3", 211, 333),
                                     ("cfg1", 3, 500), ("cfg2", 97, 161)])
def test_kernels_agree_bitwise(gpu, cfg, H, W):
    """Kernel 2 (warp-specialised, BF_KERNEL=ws) and kernel 1 (barrier intervals, BF_KERNEL=band)
    perform the same exact integer arithmetic with different schedules and walker segmentations:
    their outputs must be bitwise equal (a synchronisation race would show). Kernel 2b (ws2)
    accumulates num / den per horizontal box without kernels 1/2's rounded F, so it agrees with
    them to that rounding (well inside the tolerance) and is checked against the oracle."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, op = make_plans(pkg, config_params(spec), img.dtype)
    outs = {}
    for k in ("band", "ws", "ws2"):
        outs[k] = run_gpu(pkg, torch, gp, img, kernel=k)
    assert np.array_equal(outs["band"], outs["ws"])
    assert_close(outs["band"], outs["ws2"], spec.intensity_max, cfg)
    assert_parity(outs["ws2"], bf.bf_box(img, op), spec.intensity_max, cfg)


@pytest.mark.parametrize("cfg,H,W,over", [("cfg1", 140, 300, {"range_kind": "tukey", "sigma_r": 40.0, "n_terms": 12}),
                                          ("cfg0", 120, 250, {"range_kind": "tukey", "sigma_r": 40.0, "n_terms": 13}),
                                          ("cfg2", 150, 330, {"n_terms": 5})])
def test_kernels_agree_nonconsecutive_and_partial(gpu, cfg, H, W, over):
    """Tukey plans select non-consecutive k (the CONSEC = false instantiations, a runtime
    recurrence step count per term) and N_eff < MAXK leaves a partial channel group (FULL =
    false): kernels 1 and 2 agree bitwise there too, kernel 2b to F's rounding, and all match
    the oracle."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, op = make_plans(pkg, config_params(spec), img.dtype, **over)
    if over.get("range_kind") == "tukey":
        ks = gp.info()["k"]
        assert any(b - a > 1 for a, b in zip(ks, ks[1:])), ks
    outs = {}
    for k in ("band", "ws", "ws2"):
        outs[k] = run_gpu(pkg, torch, gp, img, kernel=k)
    assert np.array_equal(outs["band"], outs["ws"])
    assert_close(outs["band"], outs["ws2"], spec.intensity_max, cfg)
    assert_parity(outs["ws2"], bf.bf_box(img, op), spec.intensity_max, cfg)


def test_multi_plan_case1_shared_channels(gpu):
    """bf_apply_multi (Case 1 of P:1200-1219): several range kernels over one pass of shared
    box-filtered channels. Each plan's image matches the oracle of that plan (and the plan's own
    bf_apply within the tolerance: the combine weights are scaled for the set, not bitwise)."""
    pkg, torch = gpu
    spec = CONFIGS["cfg1"]
    img = config_input(spec, H=150, W=233)
    base = config_params(spec)
    variants = [dict(sigma_r=10.0), dict(sigma_r=20.0), dict(sigma_r=45.0), dict(range_kind="tukey", sigma_r=40.0)]
    plans, refs = [], []
    for v in variants:
        gp, op = make_plans(pkg, base, img.dtype, **v)
        plans.append(gp)
        refs.append(bf.bf_box(img, op))
    t = torch.from_numpy(img).cuda()
    outs = pkg.bilateral_filter_multi(plans, t).cpu().numpy().astype(np.float64)
    for q, (gp, ref) in enumerate(zip(plans, refs)):
        assert_parity(outs[q], ref, 255.0, f"plan {q}")
        assert_parity(outs[q], run_gpu(pkg, torch, gp, img), 255.0, f"plan {q} vs bf_apply")
    # plans must share the spatial plan
    other, _ = make_plans(pkg, base, img.dtype, sigma_s=5.0)
    with pytest.raises(pkg.BFError):
        pkg.bilateral_filter_multi([plans[0], other], t)


@pytest.mark.parametrize("cfg,H,W", [("cfg0", 300, 256), ("cfg2", 260, 300), ("cfg3", 200, 240),
                                     ("cfg4", 420, 300)])
@pytest.mark.parametrize("kernel", ["band", "ws", "ws2"])
def test_sliding_sums_are_exact(gpu, cfg, H, W, kernel):
    """The vertical state slides by adding the quantised enter taps and subtracting the leave
    taps, which must cancel EXACTLY (the leave tap regenerates bit for bit what the enter tap, or
    the band's initial sum, added). Every band restarts from a fresh initial sum, so the output
    may not depend on the band height: 16-row bands and one band over the whole image must agree
    bitwise (a one-ulp mismatch in any tap would drift and show here)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp, _ = make_plans(pkg, config_params(spec), img.dtype)
    outs = []
    for th in (16, H):
        outs.append(run_gpu(pkg, torch, gp, img, kernel=kernel, band_rows=th))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("cfg,H,W,over", [("cfg0", 160, 230, {}), ("cfg3", 120, 260, {}),
                                          ("cfg0", 100, 140, {"range_kind": "tukey", "sigma_r": 40.0}),
                                          ("cfg0", 70, 90, {"n_terms": 3})])
def test_literal_window_parity(gpu, cfg, H, W, over):
    """NEXT f1, the paper's literal 3-D box filter (window [I(x) - T_r, I(x) + T_r]) on u8 images:
    the level-count kernel against the oracle's dimension-promoted evaluation of the same plan;
    integer counts make the result independent of the band height (bitwise)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    p = dict(config_params(spec))
    p.update(over)
    img = config_input(spec, H=H, W=W)
    gp = pkg.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                  radius=p["radius"], n_terms=p["n_terms"], input_dtype="u8", range_window="literal")
    op = fit.make_literal_plan(**p)
    Tr = fit.truncation_radius(p["range_kind"], p["sigma_r"])
    ref = bf.bf_promoted(img.astype(np.float64), op, Tr)[0]
    got = run_gpu(pkg, torch, gp, img)
    assert_parity(got, ref, 255.0, f"{cfg} literal {over}")
    assert np.array_equal(run_gpu(pkg, torch, gp, img, band_rows=16), got)


@pytest.mark.parametrize("cfg,over", [("cfg1", {"sigma_r": 10.0}), ("cfg0", {"sigma_r": 10.0, "n_terms": 12}),
                                      ("cfg2", {"sigma_r": 0.04, "n_terms": 16})])
def test_narrow_range_kernels(gpu, cfg, over):
    """Narrow range kernels keep many slowly decaying terms, the numerically hardest case for the
    channel recurrences (a Chebyshev recurrence measured 3.6e-3 at sigma_r = 10 in emulation and
    was rejected, tools/numerics_v6.py; the rotation recurrence stays within the tolerance)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=150, W=233)
    gp, op = make_plans(pkg, config_params(spec), img.dtype, **over)
    assert_parity(run_gpu(pkg, torch, gp, img), bf.bf_box(img, op), spec.intensity_max, f"{cfg} {over}")


@pytest.mark.parametrize("cfg,H,W,n_spatial,levels", [
    ("cfg0", 150, 230, 13, 4),      # rank 3: three separable passes (fp64 workspace)
    ("cfg0", 140, 200, 25, 4),      # rank 4
    ("cfg1", 130, 260, 25, 4),
    ("cfg0", 130, 170, 16, 4),      # a split tie group: asymmetric kernel, box pieces
    ("cfg0", 120, 150, 49, 4),      # rank 5, 15 passes
    ("cfg2", 150, 260, 13, 4),      # f32, D = 1
    ("cfg0", 160, 230, 64, 2),      # J = 2: separable with four boxes per axis (Form 4, one pass)
    ("cfg4", 230, 300, 5, 4),       # rank 2 at r = 192: the box-pair kernel cannot run it -> 2 passes
])
def test_general_spatial_plans(gpu, cfg, H, W, n_spatial, levels):
    """NEXT f3 (richer spatial plans, Table II): N_s beyond the separable
    N_s = 9 and the rank-2 N_s = 5 plans, evaluated as the exact rank factorisation's separable
    passes (num / den summed in fp64), against the oracle's direct box list on every pixel (no
    conditioning mask: ill-conditioned pixels go through the fp64 repair pass)."""
    pkg, torch = gpu
    spec = CONFIGS[cfg]
    img = config_input(spec, H=H, W=W)
    gp_l = pkg.Plan(spatial=spec.spatial, range_kind=spec.range_kind, sigma_s=spec.sigma_s, sigma_r=spec.sigma_r,
                    radius=spec.radius, n_terms=spec.n_terms, intensity_max=spec.intensity_max, n_spatial=n_spatial,
                    haar_levels=levels, input_dtype="u8" if img.dtype == np.uint8 else "f32")
    op = fit.make_plan(**dict(config_params(spec), n_spatial=n_spatial, haar_levels=levels))
    got = run_gpu(pkg, torch, gp_l, img)
    assert_parity(got, bf.bf_box(img, op), spec.intensity_max, f"{cfg} N_s={n_spatial} J={levels}")
    # band height independence (every pass restarts its exact sliding sums)
    assert np.array_equal(got, run_gpu(pkg, torch, gp_l, img, band_rows=16))
