"""Pins for the oracle evaluator (oracle/bf.py): SAT exactness, the algebraic identity with the
direct double loop (P1), the dimension-promoted 3-D form (P2), invariants (P3), the range-error
bound against the exact BF (P4), convergence (P5). No GPU."""
import math

import numpy as np
import pytest

from oracle import bf, fit
from synth import CONFIGS, config_input, config_params


def small_plan(cfg, **over):
    p = config_params(CONFIGS[cfg])
    p.update(over)
    return fit.make_plan(**p), p


# ------------------------------------------------------------------ SAT

def test_sat_examples():
    S = bf.sat2d(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert S[2, 2] == 10.0 and S[0].sum() == 0 and S[:, 0].sum() == 0      # corner total, guards
    assert bf.region_sum(S, 1, 2, 1, 2) == 4.0                              # single pixel (x,y)=(1,1)
    assert bf.region_sum(S, 1, 1, 0, 2) == 0.0                              # empty region
    ones = bf.sat2d(np.ones((5, 7)))
    yy, xx = np.indices((6, 8))
    assert np.array_equal(ones, (yy * xx).astype(float))                   # area


def test_sat_exact_on_integers():
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (23, 31)).astype(np.float64)
    S = bf.sat2d(img)
    for y in range(24):
        for x in range(32):
            assert S[y, x] == img[:y, :x].sum()


def test_box_sum_clipped_matches_loops():
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (9, 11)).astype(np.float64)
    S = bf.sat2d(img)
    for _ in range(40):
        u0, v0 = rng.integers(-12, 12, 2)
        u1, v1 = u0 + rng.integers(0, 8), v0 + rng.integers(0, 8)
        got = bf.box_sum(S, u0, u1, v0, v1)
        for y in range(9):
            for x in range(11):
                ref = sum(img[yy, xx] for yy in range(y + v0, y + v1 + 1) for xx in range(x + u0, x + u1 + 1)
                          if 0 <= yy < 9 and 0 <= xx < 11)
                assert got[y, x] == ref


# ------------------------------------------------------------------ P1 / P2

@pytest.mark.parametrize("cfg,H,W,over", [
    ("cfg0", 33, 41, {}),
    ("cfg3", 29, 37, {}),                                     # box K_s
    ("cfg1", 40, 35, {"radius": 12}),
    ("cfg2", 36, 30, {"radius": 7}),                          # D = 1, float inputs
    ("cfg4", 30, 34, {"radius": 9, "sigma_s": 3.0}),          # Tukey, non-consecutive k
    ("cfg0", 25, 27, {"n_spatial": 5}),                       # the paper's 3-box plan (rank 2)
])
def test_p1_box_evaluation_equals_direct_double_loop(cfg, H, W, over):
    plan, _ = small_plan(cfg, **over)
    I = config_input(CONFIGS[cfg], H=H, W=W)
    out, num, den, _ = bf.bf_box(I, plan, return_parts=True)
    o2, n2, d2 = bf.bf_direct(I, plan)
    scale = np.max(np.abs(den))
    assert np.max(np.abs(den.ravel() - d2)) < 1e-11 * scale
    assert np.max(np.abs(num.ravel() - n2)) < 1e-11 * scale * plan.D
    assert np.max(np.abs(out.ravel() - o2)) < 1e-9 * plan.D


def test_p2_dimension_promoted_equals_2d_when_window_covers_range():
    plan, _ = small_plan("cfg0", radius=3)
    I = config_input(CONFIGS["cfg0"], H=10, W=12)
    ob = bf.bf_box(I, plan)
    op, _, _ = bf.bf_promoted(I, plan, half_window=255.0)
    assert np.max(np.abs(ob - op)) < 1e-9


def test_p2_narrow_window_differs():
    """With a window narrower than the intensity range the literal 3-D form is a different
    filter (NEXT f1); the pin above is therefore not vacuous."""
    plan, _ = small_plan("cfg0", radius=3)
    I = config_input(CONFIGS["cfg0"], H=10, W=12)
    op, _, _ = bf.bf_promoted(I, plan, half_window=20.0)
    assert np.max(np.abs(bf.bf_box(I, plan) - op)) > 1e-3


# ------------------------------------------------------------------ P3 invariants

def test_constant_image_maps_to_itself():
    plan, _ = small_plan("cfg0")
    I = np.full((21, 19), 137.0)
    assert np.max(np.abs(bf.bf_box(I, plan) - 137.0)) < 1e-10


def test_radius_zero_is_identity():
    plan, _ = small_plan("cfg1", radius=0)
    I = config_input(CONFIGS["cfg1"], H=17, W=23)
    assert np.max(np.abs(bf.bf_box(I, plan) - I)) < 1e-9


def test_infinite_sigma_r_is_plain_spatial_filter():
    plan, _ = small_plan("cfg0", sigma_r=math.inf)
    assert plan.rng.k == [0]
    I = config_input(CONFIGS["cfg0"], H=24, W=26).astype(np.float64)
    Ks = fit.spatial_kernel_values(plan.sp)
    r = plan.radius
    ref = np.empty_like(I)
    for y in range(I.shape[0]):
        for x in range(I.shape[1]):
            ya, yb, xa, xb = max(0, y - r), min(I.shape[0], y + r + 1), max(0, x - r), min(I.shape[1], x + r + 1)
            w = Ks[ya - y + r:yb - y + r, xa - x + r:xb - x + r]
            ref[y, x] = np.sum(w * I[ya:yb, xa:xb]) / np.sum(w)
    assert np.max(np.abs(bf.bf_box(I, plan) - ref)) < 1e-10


def test_intensity_flip_and_transpose_symmetry():
    plan, _ = small_plan("cfg0")
    I = config_input(CONFIGS["cfg0"], H=26, W=26).astype(np.float64)
    out = bf.bf_box(I, plan)
    assert np.max(np.abs(bf.bf_box(255.0 - I, plan) - (255.0 - out))) < 1e-9
    assert np.max(np.abs(bf.bf_box(I.T, plan) - out.T)) < 1e-9


def test_scale_law_links_unit_and_byte_ranges():
    """s * BF_{sigma_r, D}(I) = BF_{s sigma_r, s D}(s I): cfg2's [0,1] data vs a [0,255] copy."""
    p1, _ = small_plan("cfg2", radius=6)
    p255, _ = small_plan("cfg2", radius=6, sigma_r=0.1 * 255, intensity_max=255.0)
    I = config_input(CONFIGS["cfg2"], H=25, W=22).astype(np.float64)
    assert p1.rng.k == p255.rng.k
    assert np.max(np.abs(255.0 * bf.bf_box(I, p1) - bf.bf_box(255.0 * I, p255))) < 1e-8


@pytest.mark.parametrize("cfg", ["cfg0", "cfg3", "cfg4"])
def test_local_min_max_with_slack(cfg):
    """out in [m - (M-m) rho, M + (M-m) rho] with rho = sum of negative weights / sum of weights
    over the window; strict (rho = 0) where all effective weights are non-negative."""
    over = {"radius": 6, "sigma_s": 2.0} if cfg == "cfg4" else {}
    plan, _ = small_plan(cfg, **over)
    I = config_input(CONFIGS[cfg], H=20, W=21).astype(np.float64)
    out = bf.bf_box(I, plan)
    Ks = fit.spatial_kernel_values(plan.sp)
    r = plan.radius
    for y in range(I.shape[0]):
        for x in range(I.shape[1]):
            ya, yb, xa, xb = max(0, y - r), min(I.shape[0], y + r + 1), max(0, x - r), min(I.shape[1], x + r + 1)
            win = I[ya:yb, xa:xb]
            w = Ks[ya - y + r:yb - y + r, xa - x + r:xb - x + r] * fit.range_kernel_approx(plan.rng, I[y, x] - win)
            rho = -w[w < 0].sum() / w.sum()
            m, M = win.min(), win.max()
            assert m - (M - m) * rho - 1e-9 <= out[y, x] <= M + (M - m) * rho + 1e-9


def test_fallback_on_nonpositive_denominator():
    I = np.array([[3.0, 4.0]])
    out, fb = bf.normalise(I, np.array([[1.0, 2.0]]), np.array([[0.0, -1.0]]))
    assert np.array_equal(out, I) and fb.all()


# ------------------------------------------------------------------ P4 / P5 vs the exact BF

def test_p4_range_error_bound():
    """|BF(K~_s, K~_r) - BF(K~_s, K_r)| <= D delta_r sum|K~_s| / den(x) with
    delta_r = sup_{|t|<=D} |K~_r(t) - K_r(t)| (range-only error of the N-term fit)."""
    plan, p = small_plan("cfg0", radius=5)
    I = config_input(CONFIGS["cfg0"], H=18, W=20).astype(np.float64)
    t = np.linspace(-255, 255, 20001)
    delta = np.max(np.abs(fit.range_kernel_approx(plan.rng, t) - fit.range_kernel("gaussian", 30.0)(t)))
    Ks = fit.spatial_kernel_values(plan.sp)
    ref = bf.bf_bruteforce(I, Ks, fit.range_kernel("gaussian", 30.0))
    out, num, den, _ = bf.bf_box(I, plan, return_parts=True)
    bound = 255.0 * delta * np.abs(Ks).sum() / den
    assert np.all(np.abs(out - ref) <= bound + 1e-12)
    assert delta < 1e-2


def test_p5_convergence_with_more_terms():
    I = config_input(CONFIGS["cfg3"], H=30, W=30).astype(np.float64)
    errs = []
    for N in (6, 10, 16, 24):
        plan, p = small_plan("cfg3", n_terms=N)
        ref = bf.bf_exact(I, **p)
        errs.append(bf.psnr(bf.bf_box(I, plan), ref))
    assert errs == sorted(errs) and errs[-1] > 100.0


def test_accuracy_against_exact_bf_cfg0():
    """Total approximation error of the default plan vs the exact Gaussian BF (context: the
    paper reports 38.97-44.53 dB for its literal variant)."""
    plan, p = small_plan("cfg0")
    I = config_input(CONFIGS["cfg0"], H=40, W=40)
    assert bf.psnr(bf.bf_box(I, plan), bf.bf_exact(I, **p)) > 40.0



@pytest.mark.parametrize("cfg", ["cfg0", "cfg3"])
def test_p2_literal_window_equals_windowed_double_loop(cfg):
    """NEXT f1 pin: the literal dimension-promoted evaluation (per-level 2-D box sums, z-window
    [I(x) - T_r, I(x) + T_r] with a 1-D SAT along z) equals the direct double loop of
    sum_y K~_s K~_r(I(x)-I(y)) B(I(x)-I(y)) I(y) / sum(...) with B the window box
    on an integer image: two different evaluations of the same definition."""
    spec = CONFIGS[cfg]
    p = config_params(spec)
    I = config_input(spec, H=30, W=37).astype(np.float64)
    plan = fit.make_literal_plan(**p)
    Tr = fit.truncation_radius(p["range_kind"], p["sigma_r"])
    assert Tr < 255.0 and abs(plan.D - Tr) < 1e-12
    out, num, den = bf.bf_promoted(I, plan, Tr)
    o2, n2, d2 = bf.bf_direct(I, plan, window=Tr)
    scale = np.max(np.abs(d2))
    assert np.max(np.abs(den.ravel() - d2)) <= 1e-10 * scale
    assert np.max(np.abs(num.ravel() - n2)) <= 1e-10 * scale * 255
    assert np.max(np.abs(out.ravel() - o2)) <= 1e-8
    # the window matters: without it the same cosine series gives a different filter
    o3, _, _ = bf.bf_direct(I, plan)
    assert np.max(np.abs(o3 - o2)) > 1e-3


def test_literal_plan_accuracy_against_exact_bf():
    """The literal method with a handful of terms approximates the exact BF (Gaussian spatial
    kernel, range kernel truncated at T_r) far better than the T = D hot path at the same N, the
    paper's point about truncating the range kernel first."""
    spec = CONFIGS["cfg0"]
    p = dict(config_params(spec))
    p["n_terms"] = 4
    I = config_input(spec, H=40, W=48).astype(np.float64)
    exact = bf.bf_exact(I, **p)
    lit = bf.bf_promoted(I, fit.make_literal_plan(**p), fit.truncation_radius("gaussian", p["sigma_r"]))[0]
    full = bf.bf_box(I, fit.make_plan(**p))
    e_lit = np.sqrt(np.mean((lit - exact) ** 2))
    e_full = np.sqrt(np.mean((full - exact) ** 2))
    assert e_lit < 0.5 * e_full
