"""Oracle fitter: range cosine coefficients, 2-D Haar coefficients, best-N selection, lowering.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). fp64 throughout. "P:n" = PAPER.md line n.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------------------------
# Kernels K_r / K_s (symmetric, decreasing on R+).
# --------------------------------------------------------------------------------------------


def range_kernel(kind: str, sigma: float):
    """K_r as a vectorised function of t.

    gaussian: G_sigma(t) = exp(-t^2 / 2 sigma^2); sigma = +inf gives K_r == 1.
    tukey:    (1 - (t/s)^2)^2 for |t| <= s, else 0 (Tukey biweight with scale s, BASELINE cfg4;
              SURVEY Q22).
    """
    if kind == "gaussian":
        if math.isinf(sigma):
            return lambda t: np.ones_like(np.asarray(t, dtype=np.float64))
        return lambda t: np.exp(-np.asarray(t, dtype=np.float64) ** 2 / (2.0 * sigma * sigma))
    if kind == "tukey":
        def f(t):
            t = np.asarray(t, dtype=np.float64)
            u = t / sigma
            return np.where(np.abs(u) <= 1.0, (1.0 - u * u) ** 2, 0.0)
        return f
    raise ValueError(f"unknown range kernel {kind!r}")


def range_kernel_kinks(kind: str, sigma: float) -> list:
    """Points where K_r is not smooth (quadrature panels are split there)."""
    return [-sigma, sigma] if kind == "tukey" else []


def truncation_radius(kind: str, sigma: float, eps: float = 0.01) -> float:
    """T = K^{-1}(eps) (eps = 0.01 "a reasonable value"). Used only for the literal
    [-T_r, T_r] fit (Table V pin, NEXT f1); the hot path uses T = D."""
    if kind == "gaussian":
        return sigma * math.sqrt(-2.0 * math.log(eps))
    if kind == "tukey":
        return sigma * math.sqrt(1.0 - math.sqrt(eps))
    raise ValueError(kind)


# --------------------------------------------------------------------------------------------
# Range fit: truncated trigonometric functions on [-T, T].
#   a_0 = 1/(2T) int_{-T}^{T} f,  a_j = 1/T int_{-T}^{T} f(x) cos(pi j x / T) dx,  b_j = 0.
# --------------------------------------------------------------------------------------------

_GL_ORDER = 16
_GL_X, _GL_W = np.polynomial.legendre.leggauss(_GL_ORDER)


def _gl_nodes(a: float, b: float, breakpoints: list, n_panels: int):
    """Composite Gauss-Legendre nodes/weights on [a, b], panels split at `breakpoints`."""
    cuts = sorted({a, b, *[p for p in breakpoints if a < p < b]})
    xs, ws = [], []
    total = b - a
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        m = max(1, int(math.ceil(n_panels * (hi - lo) / total)))
        edges = np.linspace(lo, hi, m + 1)
        for e0, e1 in zip(edges[:-1], edges[1:]):
            half = 0.5 * (e1 - e0)
            xs.append(0.5 * (e0 + e1) + half * _GL_X)
            ws.append(half * _GL_W)
    return np.concatenate(xs), np.concatenate(ws)


def range_coefficients(kind: str, sigma: float, T: float, M: int, truncate_at: float | None = None) -> np.ndarray:
    """Cosine coefficients a_0..a_{M-1} of K_r on [-T, T].

    If `truncate_at` is given, the truncated kernel K_r^T (zero outside [-truncate_at,
    truncate_at]) is expanded instead of K_r itself. The hot path expands K_r on
    [-D, D] without truncation (Case 1).

    The integrals are evaluated by composite Gauss-Legendre quadrature (16 nodes per panel,
    >= 2 panels per cosine period, panels split at the kernel's kinks) - never adaptive
    quadrature.
    """
    f = range_kernel(kind, sigma)
    kinks = list(range_kernel_kinks(kind, sigma))
    if truncate_at is not None:
        kinks += [-truncate_at, truncate_at]
    n_panels = 2 * M + 64
    x, w = _gl_nodes(-T, T, kinks, n_panels)
    fx = f(x)
    if truncate_at is not None:
        fx = np.where(np.abs(x) <= truncate_at, fx, 0.0)
    a = np.empty(M)
    a[0] = np.sum(w * fx) / (2.0 * T)
    for j in range(1, M):
        a[j] = np.sum(w * fx * np.cos(math.pi * j * x / T)) / T
    return a


def select_best_n(coeffs: np.ndarray, N: int, rel_tie: float = 1e-12, rel_zero: float = 1e-14) -> list:
    """Best N-term selection: the N largest |c| among the given candidates,
    which are in canonical order. Ties (|c_i| == |c_j| within `rel_tie`
    relative) go to the smaller canonical index; coefficients with
    |c| <= rel_zero * max|c| are pruned, so fewer than N may be returned.
    Returns the selected canonical indices in canonical order."""
    mag = np.abs(np.asarray(coeffs, dtype=np.float64))
    cmax = float(mag.max()) if mag.size else 0.0
    if cmax == 0.0:
        return []
    alive = [i for i in range(mag.size) if mag[i] > rel_zero * cmax]
    if len(alive) <= N:
        return sorted(alive)
    by_mag = sorted(alive, key=lambda i: (-mag[i], i))
    vN = mag[by_mag[N - 1]]
    sure = [i for i in alive if mag[i] > vN * (1.0 + rel_tie)]
    ties = sorted(i for i in alive if vN * (1.0 - rel_tie) <= mag[i] <= vN * (1.0 + rel_tie))
    chosen = sure + ties[: N - len(sure)]
    return sorted(chosen)


@dataclass
class RangePlan:
    """Lambda^r = {(k, a_k)} on [-T, T]."""
    kind: str
    sigma: float
    T: float
    M: int
    k: list
    a: list
    all_a: np.ndarray = field(repr=False, default=None)


def fit_range(kind: str, sigma: float, D: float, N: int, m_factor: int = 20) -> RangePlan:
    """Hot-path range plan: K_r expanded on [-D, D] (T = T_{r_i} := D; SURVEY
    Q1/Q2), candidates k < M = m_factor * N, best N by raw |a_k|."""
    M = m_factor * N
    a = range_coefficients(kind, sigma, D, M)
    sel = select_best_n(a, N)
    return RangePlan(kind, sigma, D, M, sel, [float(a[i]) for i in sel], a)


# --------------------------------------------------------------------------------------------
# Spatial fit: 2-D Haar functions on [-T_s, T_s]^2.
# --------------------------------------------------------------------------------------------

PHI = ("phi",)


def haar_index_1d(J: int) -> list:
    """1-D Haar functions in canonical order: phi first, then psi_{j,k} by (j, k).
    Level 0 is the single mother function psi_{0,0}; level j >= 1 has
    k in K_j = {-2^{j-1}, ..., -1, 1, ..., 2^{j-1}}."""
    idx = [PHI, ("psi", 0, 0)]
    for j in range(1, J + 1):
        h = 2 ** (j - 1)
        idx += [("psi", j, k) for k in list(range(-h, 0)) + list(range(1, h + 1))]
    return idx


def haar_cells(h, T: float) -> list:
    """Support cells of a 1-D Haar function as [(lo, hi, sign)] (Appendix A):
    phi = +1 on A = [-T, T]; psi_{j,k} = +1 on A1 = [2^-j (Z-T), 2^-j Z) and -1 on
    A2 = [2^-j Z, 2^-j (Z+T)], Z_k = sign(k)(2|k|-1)T (eq:Haar_set)."""
    if h[0] == "phi":
        return [(-T, T, 1.0)]
    _, j, k = h
    Z = 0.0 if k == 0 else math.copysign((2 * abs(k) - 1) * T, k)
    s = 2.0 ** (-j)
    return [(s * (Z - T), s * Z, 1.0), (s * Z, s * (Z + T), -1.0)]


def _gauss_integral(sigma: float, lo: float, hi: float) -> float:
    """int_lo^hi exp(-x^2 / 2 sigma^2) dx (closed form via erf)."""
    c = sigma * math.sqrt(2.0)
    return sigma * math.sqrt(math.pi / 2.0) * (math.erf(hi / c) - math.erf(lo / c))


def spatial_factor_integral(kind: str, sigma: float, lo: float, hi: float) -> float:
    """int_lo^hi g(x) dx for the 1-D factor g of a separable K_s on the square:
    gaussian g = exp(-x^2/2 sigma^2) (K_s(||x||) = g(x) g(y)); box g = 1."""
    if kind == "gaussian":
        return _gauss_integral(sigma, lo, hi)
    if kind == "box":
        return hi - lo
    raise ValueError(kind)


def haar_coefficient_1d(kind: str, sigma: float, T: float, h) -> float:
    """c_0 = (1/2T) int g phi;  c_{jk} = (2^j / 2T) int g psi_{j,k}."""
    norm = 1.0 if h[0] == "phi" else 2.0 ** h[1]
    tot = sum(sgn * spatial_factor_integral(kind, sigma, lo, hi) for lo, hi, sgn in haar_cells(h, T))
    return norm * tot / (2.0 * T)


def family(a, b) -> int:
    """Family of phi/psi products in the order of eq:Haar_expansion:
    0 phi(x)phi(y), 1 phi(x)psi(y), 2 psi(x)phi(y), 3 psi(x)psi(y)."""
    return (0 if a == PHI else 2) + (0 if b == PHI else 1)


def _h_key(h):
    return (-1, 0) if h == PHI else (h[1], h[2])


def canonical_key(a, b):
    """(family, j1, k1, j2, k2) canonical order."""
    return (family(a, b), *_h_key(a), *_h_key(b))


@dataclass
class SpatialPlan:
    """Lambda^s: selected 2-D Haar terms, their coefficients, and the lowered
    integer-offset boxes (u0, u1, v0, v1, weight) with u = column offset, v = row offset."""
    kind: str
    sigma: float
    radius: int
    T: float
    terms: list            # [(a, b, c)] in canonical order; a = x factor, b = y factor
    boxes: list            # [(u0, u1, v0, v1, w)] inclusive integer ranges
    all_terms: list = field(repr=False, default=None)


def haar_coefficients_2d(kind: str, sigma: float, T: float, J: int) -> list:
    """All 2-D coefficients with levels <= J (eq:Haar_2D_coefficients).

    K_s on the square is separable, K_s(x, y) = g(x) g(y), so each 2-D integral
    (n_a n_b / 4T^2) int int g(x) g(y) h_a(x) h_b(y) dx dy factors (Fubini) into the product
    of the 1-D integrals (n_a/2T) int g h_a * (n_b/2T) int g h_b (pinned against 2-D
    quadrature in tests)."""
    idx = haar_index_1d(J)
    c1 = {h: haar_coefficient_1d(kind, sigma, T, h) for h in idx}
    out = [(a, b, c1[a] * c1[b]) for a in idx for b in idx]
    out.sort(key=lambda t: canonical_key(t[0], t[1]))
    return out


def discretize(lo: float, hi: float) -> tuple:
    """Integer offsets u with lo <= u < hi (half-open pixel cells)."""
    return int(math.ceil(lo)), int(math.ceil(hi)) - 1


def lower_to_boxes(terms: list, T: float) -> list:
    """Appendix A: phi phi -> 1 box, phi psi / psi phi -> 2 boxes with signs
    (+, -), psi psi -> 4 boxes (+ - + -) on A1xA1, A1xA2, A2xA2, A2xA1 (eq:2D_box_N_terms);
    each weighted by its coefficient c_j (eq:Box_N_terms). Empty boxes are dropped."""
    boxes = []
    for a, b, c in terms:
        for xlo, xhi, sx in haar_cells(a, T):
            for ylo, yhi, sy in haar_cells(b, T):
                u0, u1 = discretize(xlo, xhi)
                v0, v1 = discretize(ylo, yhi)
                if u1 >= u0 and v1 >= v0:
                    boxes.append((u0, u1, v0, v1, c * sx * sy))
    return boxes


def fit_spatial(kind: str, sigma: float, radius: int, n_spatial: int, J: int = 4) -> SpatialPlan:
    """Best N_s-term 2-D Haar approximation of the truncated K_s on
    [-T_s, T_s]^2 with T_s = r + 1/2, levels <= J, lowered to boxes."""
    T = radius + 0.5
    allt = haar_coefficients_2d(kind, sigma, T, J)
    sel = select_best_n(np.array([t[2] for t in allt]), n_spatial)
    terms = [allt[i] for i in sel]
    return SpatialPlan(kind, sigma, radius, T, terms, lower_to_boxes(terms, T), allt)


# --------------------------------------------------------------------------------------------
# The complete plan (the oracle's counterpart of bf_plan_create).
# --------------------------------------------------------------------------------------------


@dataclass
class Plan:
    rng: RangePlan
    sp: SpatialPlan
    D: float

    @property
    def radius(self) -> int:
        return self.sp.radius


def make_plan(spatial: str, range_kind: str, sigma_s: float, sigma_r: float, radius: int,
              n_terms: int, intensity_max: float = 255.0, n_spatial: int = 9,
              m_factor: int = 20, haar_levels: int = 4, **_ignored) -> Plan:
    rng = fit_range(range_kind, sigma_r, intensity_max, n_terms, m_factor)
    sp = fit_spatial(spatial, sigma_s, radius, n_spatial, haar_levels)
    return Plan(rng, sp, float(intensity_max))


def make_literal_plan(spatial: str, range_kind: str, sigma_s: float, sigma_r: float, radius: int,
                      n_terms: int, n_spatial: int = 9, m_factor: int = 20, **_ignored) -> Plan:
    """The paper-literal range plan (NEXT f1): T = T_r = K_r^{-1}(0.01), the cosine
    basis of period 2 T_r fitted on [-T_r, T_r]; Plan.D = T_r is then the period
    half-width the channels use (P:468 with T_r). Evaluate with bf.bf_promoted(I, plan, T_r)."""
    Tr = truncation_radius(range_kind, sigma_r)
    return make_plan(spatial, range_kind, sigma_s, sigma_r, radius, n_terms, intensity_max=Tr,
                     n_spatial=n_spatial, m_factor=m_factor)


def spatial_kernel_values(sp: SpatialPlan) -> np.ndarray:
    """K~_s(u, v) on the (2r+1)^2 integer grid from the lowered boxes (eq:Box_N_terms);
    array indexed [v + r, u + r] (row offset, column offset)."""
    r = sp.radius
    K = np.zeros((2 * r + 1, 2 * r + 1))
    for u0, u1, v0, v1, w in sp.boxes:
        K[v0 + r:v1 + r + 1, u0 + r:u1 + r + 1] += w
    return K


def range_kernel_approx(rp: RangePlan, t) -> np.ndarray:
    """K~_r(t) = sum_{k in Lambda^r} a_k cos(pi k t / T) (eq:trigonometric_N_terms)."""
    t = np.asarray(t, dtype=np.float64)
    out = np.zeros_like(t)
    for k, a in zip(rp.k, rp.a):
        out = out + a * np.cos(math.pi * k * t / rp.T)
    return out
