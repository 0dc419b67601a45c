"""Pins for the oracle fitter (oracle/fit.py) against things other than itself:
closed forms, independent quadrature, the L2-projection identity of a complete Haar system, and
the paper's Table V range row. No GPU."""
import math
import os

import numpy as np
import pytest
from scipy import integrate

from oracle import fit

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ range fit

def gaussian_ak_infinite(k, sigma, D):
    """int_{-inf}^{inf} exp(-t^2/2s^2) cos(w t) dt = s sqrt(2 pi) exp(-w^2 s^2 / 2); valid on
    [-D, D] when exp(-D^2 / 2 s^2) is negligible."""
    w = math.pi * k / D
    full = sigma * math.sqrt(2 * math.pi) * math.exp(-(w * sigma) ** 2 / 2)
    return full / (2 * D) if k == 0 else full / D


@pytest.mark.parametrize("sigma,D,N", [(30.0, 255.0, 8), (20.0, 255.0, 12), (0.1, 1.0, 16), (15.0, 255.0, 10)])
def test_gaussian_coefficients_closed_form(sigma, D, N):
    a = fit.range_coefficients("gaussian", sigma, D, 20 * N)
    ref = np.array([gaussian_ak_infinite(k, sigma, D) for k in range(20 * N)])
    assert np.max(np.abs(a - ref)) < 1e-13


def test_gaussian_coefficients_wide_kernel_independent_quadrature():
    # sigma comparable to D: truncation at +-D matters, compare against scipy quad (low k only).
    sigma, D = 200.0, 255.0
    a = fit.range_coefficients("gaussian", sigma, D, 20)
    for k in range(6):
        v, _ = integrate.quad(lambda t: math.exp(-t * t / (2 * sigma ** 2)) * math.cos(math.pi * k * t / D),
                              -D, D, epsabs=1e-13, epsrel=1e-12, limit=400)
        ref = v / (2 * D) if k == 0 else v / D
        assert abs(a[k] - ref) < 1e-12


def tukey_ak(k, s, D):
    """(1/D) int_{-s}^{s} (1 - t^2/s^2)^2 cos(pi k t / D) dt = (s/D) F(z), z = pi k s / D,
    F(z) = 16 [(3 - z^2) sin z - 3 z cos z] / z^5 (F(0) = 16/15); a_0 has the 1/(2D) factor."""
    z = math.pi * k * s / D
    if k == 0:
        return (s / (2 * D)) * 16.0 / 15.0
    if z < 0.5:
        # series of F(z) = 16/15 - 8 z^2/105 + 2 z^4/945 - ... (from the cosine Taylor series)
        F = sum((-1) ** n * z ** (2 * n) / math.factorial(2 * n) * 16.0 / ((2 * n + 1) * (2 * n + 3) * (2 * n + 5))
                for n in range(12))
    else:
        F = 16.0 * ((3 - z * z) * math.sin(z) - 3 * z * math.cos(z)) / z ** 5
    return (s / D) * F


def test_tukey_coefficients_closed_form():
    s, D, N = 40.0, 255.0, 24
    a = fit.range_coefficients("tukey", s, D, 20 * N)
    ref = np.array([tukey_ak(k, s, D) for k in range(20 * N)])
    assert np.max(np.abs(a - ref)) < 1e-13


def test_tukey_series_matches_closed_form_near_switch():
    s, D = 40.0, 255.0
    for z in (0.49, 0.51):
        k = z * D / (math.pi * s)
        # evaluate both branches at the same z through the public helper's formula
        F_series = sum((-1) ** n * z ** (2 * n) / math.factorial(2 * n) * 16.0 / ((2 * n + 1) * (2 * n + 3) * (2 * n + 5))
                       for n in range(12))
        F_closed = 16.0 * ((3 - z * z) * math.sin(z) - 3 * z * math.cos(z)) / z ** 5
        assert abs(F_series - F_closed) < 1e-10
        assert k > 0


def test_constant_kernel_is_dc_only():
    a = fit.range_coefficients("gaussian", math.inf, 255.0, 40)
    assert abs(a[0] - 1.0) < 1e-14 and np.max(np.abs(a[1:])) < 1e-13
    rp = fit.fit_range("gaussian", math.inf, 255.0, 5)
    assert rp.k == [0] and abs(rp.a[0] - 1.0) < 1e-14   # zero coefficients pruned (N_eff < N)


def test_full_cosine_series_reconstructs_kernel():
    rp = fit.range_coefficients("gaussian", 30.0, 255.0, 200)
    t = np.linspace(-255, 255, 1001)
    rec = sum(rp[k] * np.cos(math.pi * k * t / 255.0) for k in range(200))
    assert np.max(np.abs(rec - np.exp(-t * t / 1800.0))) < 1e-12


def test_selection_examples():
    assert fit.select_best_n(np.array([5.0, -7.0, 3.0]), 1) == [1]           # S:233 max magnitude
    assert fit.select_best_n(np.array([1.0, -1.0, 1.0, 0.5]), 2) == [0, 1]   # ties -> smaller index
    assert fit.select_best_n(np.array([1.0, 0.0, 1e-20, 0.3]), 4) == [0, 3]   # zeros pruned
    assert fit.select_best_n(np.array([0.2, 0.9, 0.5]), 2) == [1, 2]          # canonical order out


def test_table_v_range_row():
    """PAPER.md Table V: G_40 range kernel, N -> minimal M."""
    rows = [tuple(map(int, l.split())) for l in open(os.path.join(GOLDEN, "table5_range_row.txt"))
            if l.strip() and not l.startswith("#")]
    Tr = fit.truncation_radius("gaussian", 40.0)
    assert abs(Tr - 40.0 * math.sqrt(-2 * math.log(0.01))) < 1e-12
    a = fit.range_coefficients("gaussian", 40.0, Tr, 60, truncate_at=Tr)
    for N, M in rows:
        sel = fit.select_best_n(a, N)
        assert max(sel) + 1 == M, (N, sel)


def test_hot_path_selected_k_sets():
    """T = D reading: Gaussian picks k = 0..N-1; Tukey(40) with N = 24 picks the
    non-consecutive set the closed form ranks highest."""
    assert fit.fit_range("gaussian", 0.1, 1.0, 16).k == list(range(16))
    tk = fit.fit_range("tukey", 40.0, 255.0, 24).k
    ref = [tukey_ak(k, 40.0, 255.0) for k in range(480)]
    want = sorted(sorted(range(480), key=lambda k: -abs(ref[k]))[:24])
    assert tk == want == list(range(18)) + [20, 21, 22, 23, 27, 28]


# ------------------------------------------------------------------ spatial fit

def _pointwise_haar(h, T, x):
    """Haar function values at points x with half-open cells, written from
    eq:Haar_scaling / eq:Haar_mother / eq:Haar_set directly (not via haar_cells)."""
    x = np.asarray(x, dtype=np.float64)
    if h == fit.PHI:
        return np.where((x >= -T) & (x < T), 1.0, 0.0)
    _, j, k = h
    shift = 0.0 if k == 0 else np.sign(k) * (2 * abs(k) - 1) * T
    t = 2.0 ** j * x - shift                       # psi_{j,k}(x) = psi_00(2^j x - sign(k)(2|k|-1)T)
    return np.where((t >= -T) & (t < 0), 1.0, np.where((t >= 0) & (t < T), -1.0, 0.0))


@pytest.mark.parametrize("sigma,r", [(3.0, 9), (16.0, 48), (64.0, 192)])
def test_haar_1d_coefficients_independent_quadrature(sigma, r):
    T = r + 0.5
    for h in fit.haar_index_1d(3):
        cells = fit.haar_cells(h, T)
        v = 0.0
        for lo, hi, sgn in cells:
            q, _ = integrate.quad(lambda x: math.exp(-x * x / (2 * sigma ** 2)), lo, hi, epsabs=1e-15, epsrel=1e-13)
            v += sgn * q
        norm = 1.0 if h == fit.PHI else 2.0 ** h[1]
        assert abs(fit.haar_coefficient_1d("gaussian", sigma, T, h) - norm * v / (2 * T)) < 1e-13


def test_haar_2d_coefficients_against_2d_quadrature():
    """eq:Haar_2D_coefficients by brute-force 2-D midpoint quadrature of
    K_s(x, y) h_a(x) h_b(y) for an isotropic Gaussian K_s on the square."""
    sigma, r = 3.0, 9
    T = r + 0.5
    n = 2048          # multiple of 2^(J+1): cell edges fall between midpoints
    x = -T + (np.arange(n) + 0.5) * (2 * T / n)
    K = np.exp(-(x[:, None] ** 2 + x[None, :] ** 2) / (2 * sigma ** 2))    # [x, y]
    allt = {(a, b): c for a, b, c in fit.haar_coefficients_2d("gaussian", sigma, T, 2)}
    for a, b in [(fit.PHI, fit.PHI), (fit.PHI, ("psi", 1, 1)), (("psi", 1, -1), fit.PHI),
                 (("psi", 1, 1), ("psi", 1, -1)), (("psi", 2, 2), ("psi", 1, 1)), (("psi", 0, 0), fit.PHI)]:
        na = 1.0 if a == fit.PHI else 2.0 ** a[1]
        nb = 1.0 if b == fit.PHI else 2.0 ** b[1]
        ha = _pointwise_haar(a, T, x)
        hb = _pointwise_haar(b, T, x)
        integral = np.sum(K * ha[:, None] * hb[None, :]) * (2 * T / n) ** 2
        ref = na * nb * integral / (4 * T * T)
        assert abs(allt[(a, b)] - ref) < 2e-6, (a, b, allt[(a, b)], ref)


@pytest.mark.parametrize("sigma,r", [(3.0, 9), (16.0, 48)])
def test_complete_haar_system_gives_cell_averages(sigma, r):
    """With every 2-D term up to level J selected, the lowered boxes must reproduce the L2
    projection of K_s onto the 2^{J+1} x 2^{J+1} dyadic cells, i.e. cell averages (closed form
    via erf), at every integer offset. Pins coefficients, normalisations, signs and lowering."""
    J = 3
    T = r + 0.5
    sp = fit.fit_spatial("gaussian", sigma, r, n_spatial=10 ** 6, J=J)
    K = fit.spatial_kernel_values(sp)
    ncell = 2 ** (J + 1)
    w = 2 * T / ncell
    u = np.arange(-r, r + 1)
    cell = np.floor((u + T) / w).astype(int)
    c = sigma * math.sqrt(2)
    avg = np.array([sigma * math.sqrt(math.pi / 2) * (math.erf((-T + (i + 1) * w) / c) - math.erf((-T + i * w) / c)) / w
                    for i in range(ncell)])
    ref = np.outer(avg[cell], avg[cell])
    assert np.max(np.abs(K - ref)) < 1e-13


def test_lowering_pointwise_exact():
    """Each Haar term lowers to boxes whose sum equals c * h_a(u) h_b(v) at every integer offset."""
    r = 10
    T = r + 0.5
    u = np.arange(-r, r + 1, dtype=np.float64)
    for a, b in [(fit.PHI, ("psi", 1, -1)), (("psi", 2, -2), ("psi", 1, 1)), (("psi", 0, 0), ("psi", 3, 4))]:
        sp = fit.SpatialPlan("gaussian", 1.0, r, T, [(a, b, 0.7)], fit.lower_to_boxes([(a, b, 0.7)], T))
        K = fit.spatial_kernel_values(sp)                         # [v, u]
        ref = 0.7 * np.outer(_pointwise_haar(b, T, u), _pointwise_haar(a, T, u))
        assert np.array_equal(K, ref)


def test_box_kernel_is_one_box():
    sp = fit.fit_spatial("box", 0.0, 10, 9)
    assert len(sp.terms) == 1 and abs(sp.terms[0][2] - 1.0) < 1e-15
    assert sp.boxes == [(-10, 10, -10, 10, sp.terms[0][2])]


def test_default_nine_terms_symmetric_and_separable():
    """N_s = 9 picks phi/psi_{1,+-1} products (f1+f2+f3+f4): K~_s is symmetric and rank 1
    with a 1-D factor that is constant on |u| <= r_in = floor((2r+1)/4) and on r_in < |u| <= r."""
    for sigma, r in [(3.0, 9), (8.0, 24), (16.0, 48), (64.0, 192)]:
        sp = fit.fit_spatial("gaussian", sigma, r, 9)
        assert len(sp.terms) == 9
        assert {(fit.family(a, b)) for a, b, _ in sp.terms} == {0, 1, 2, 3}
        K = fit.spatial_kernel_values(sp)
        assert np.allclose(K, K.T, rtol=0, atol=1e-15) and np.allclose(K, K[::-1, ::-1], rtol=0, atol=1e-15)
        U, s, Vt = np.linalg.svd(K)
        assert s[1] < 1e-12 * s[0]
        f = K[r] / math.sqrt(K[r, r])
        rin = (2 * r + 1) // 4
        assert np.ptp(f[r - rin:r + rin + 1]) < 1e-12 and np.ptp(f[:r - rin]) < 1e-12


def test_spatial_selection_never_splits_tie_group():
    """Isotropic kernels give exact 4-way ties: N_s = 2..4 resolve them by canonical
    order deterministically."""
    sp = fit.fit_spatial("gaussian", 3.0, 9, 3)
    keys = [fit.canonical_key(a, b) for a, b, _ in sp.terms]
    assert keys == sorted(keys) and len(keys) == 3
    assert sp.terms[0][0] == fit.PHI and sp.terms[0][1] == fit.PHI


@pytest.mark.parametrize("kind,sigma", [("gaussian", 20.0), ("gaussian", 0.1), ("tukey", 40.0), ("tukey", 7.5)])
def test_truncation_radius_is_the_eps_level_of_the_kernel(kind, sigma):
    """T_r = K_r^{-1}(eps) (eps = 0.01): evaluated through the kernel itself, not through a
    second copy of the inverse formula: K_r(T_r) = eps and K_r decreasing through it."""
    T = fit.truncation_radius(kind, sigma)
    K = fit.range_kernel(kind, sigma)
    assert abs(float(K(T)) - 0.01) <= 1e-12
    assert float(K(0.999 * T)) > 0.01 > float(K(1.001 * T))


def test_canonical_key_orders_a_hand_written_list():
    """Canonical order: family first (phi.phi, phi(x)psi(y), psi(x)phi(y),
    psi.psi, eq:Haar_expansion P:304-307), then (j1, k1) of the x factor, then (j2, k2); phi sorts
    before every psi. The expected order is written out by hand."""
    P, s = fit.PHI, lambda j, k: ("psi", j, k)
    expected = [
        (P, P),
        (P, s(0, 0)), (P, s(1, -1)), (P, s(1, 1)), (P, s(2, -2)),
        (s(0, 0), P), (s(1, -1), P), (s(2, 1), P),
        (s(0, 0), s(0, 0)), (s(0, 0), s(1, 1)), (s(1, -1), s(0, 0)), (s(1, -1), s(2, -2)),
        (s(1, 1), s(0, 0)), (s(2, -2), s(1, -1)),
    ]
    shuffled = [expected[i] for i in (13, 2, 7, 0, 10, 5, 12, 1, 9, 3, 11, 6, 4, 8)]
    assert sorted(shuffled, key=lambda t: fit.canonical_key(*t)) == expected
