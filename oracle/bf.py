"""Oracle evaluator of the N-term bilateral-filter approximation, and the brute-force BF.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). fp64 numpy; slow; "P:n" = PAPER.md line n.

Conventions (DESIGN.md readings): images are indexed [row, col] = [y, x]; a box
(u0, u1, v0, v1, w) covers column offsets u0..u1 and row offsets v0..v1 around the output
pixel; pixels outside the image contribute 0; a non-positive or non-finite
denominator falls back to I(x).
"""
from __future__ import annotations

import math

import numpy as np

from .fit import Plan, range_kernel, range_kernel_approx, spatial_kernel_values

# --------------------------------------------------------------------------------------------
# Summed-area tables.
# --------------------------------------------------------------------------------------------


def sat2d(img: np.ndarray) -> np.ndarray:
    """2-D SAT with a zero guard row/column: S[y+1, x+1] = sum_{y'<=y, x'<=x} I.

    Built with the paper's one-pass recurrence c(x,y) = c(x,y-1) + I(x,y),
    S(x,y) = S(x-1,y) + c(x,y) (eq:sum_sat_recurrence_2D), vectorised over rows/columns."""
    H, W = img.shape
    S = np.zeros((H + 1, W + 1), dtype=np.float64)
    c = np.cumsum(np.asarray(img, dtype=np.float64), axis=0)      # c(x, y) = c(x, y-1) + I(x, y)
    S[1:, 1:] = np.cumsum(c, axis=1)                                # S(x, y) = S(x-1, y) + c(x, y)
    return S


def region_sum(S: np.ndarray, x0, x1, y0, y1):
    """S(R) for R = (x0, x1] x (y0, y1] in guard coordinates (eq:sum_sat_sum_region_2D):
    S(x1,y1) - S(x1,y0) - S(x0,y1) + S(x0,y0)."""
    return S[y1, x1] - S[y0, x1] - S[y1, x0] + S[y0, x0]


def box_sum(S: np.ndarray, u0: int, u1: int, v0: int, v1: int) -> np.ndarray:
    """For every pixel (y, x): sum of the channel over columns x+u0..x+u1, rows y+v0..y+v1,
    clipped to the image (out-of-image pixels are 0)."""
    Hp, Wp = S.shape
    H, W = Hp - 1, Wp - 1
    xs = np.arange(W)
    ys = np.arange(H)
    x0 = np.clip(xs + u0, 0, W)
    x1 = np.clip(xs + u1 + 1, 0, W)
    y0 = np.clip(ys + v0, 0, H)
    y1 = np.clip(ys + v1 + 1, 0, H)
    return region_sum(S, x0[None, :], x1[None, :], y0[:, None], y1[:, None])


def spatial_filter(X: np.ndarray, boxes: list) -> np.ndarray:
    """sum_{c_j in Lambda^s} c_j sum_{y in N^j_x} X(y) (eq:2D_box_N_terms_s) via one
    fp64 SAT of X and four references per box."""
    S = sat2d(X)
    out = np.zeros(X.shape, dtype=np.float64)
    for u0, u1, v0, v1, w in boxes:
        out += w * box_sum(S, u0, u1, v0, v1)
    return out


# --------------------------------------------------------------------------------------------
# The box-filter evaluation (eq:numerator_2D_box_N_terms with T = D).
# --------------------------------------------------------------------------------------------


def channels(I: np.ndarray, k: int, D: float):
    """g^c_k = cos(pi k I / T), g^s_k = sin(pi k I / T), G^c_k = g^c_k I, G^s_k = g^s_k I,
    with T = D."""
    I = np.asarray(I, dtype=np.float64)
    ph = math.pi * k * I / D
    gc, gs = np.cos(ph), np.sin(ph)
    return gc, gs, gc * I, gs * I


def bf_box(I: np.ndarray, plan: Plan, return_parts: bool = False):
    """Oracle output of the N-term approximation, evaluated with box filters.

    num(x) = sum_k a_k [g^c_k(x) S(G^c_k)(x) + g^s_k(x) S(G^s_k)(x)]   (eq:numerator_2D_box_N_terms,
    den(x) = sum_k a_k [g^c_k(x) S(g^c_k)(x) + g^s_k(x) S(g^s_k)(x)]    P:487-493, per-k factors Q17)
    where S is the lowered spatial box operator (eq:2D_box_N_terms_s) and the z-window sum is
    the identity because T = D covers every intensity (P:469-478 with T_{r_i} = D).
    out = num / den (eq:BF ratio); den <= 0 or non-finite -> I(x)."""
    I = np.asarray(I, dtype=np.float64)
    num = np.zeros_like(I)
    den = np.zeros_like(I)
    for k, a in zip(plan.rng.k, plan.rng.a):
        gc, gs, Gc, Gs = channels(I, k, plan.D)
        num += a * (gc * spatial_filter(Gc, plan.sp.boxes) + gs * spatial_filter(Gs, plan.sp.boxes))
        den += a * (gc * spatial_filter(gc, plan.sp.boxes) + gs * spatial_filter(gs, plan.sp.boxes))
    out, fallback = normalise(I, num, den)
    if return_parts:
        return out, num, den, fallback
    return out


def normalise(I, num, den):
    ok = np.isfinite(den) & (den > 0)
    with np.errstate(divide="ignore", invalid="ignore"):
        out = np.where(ok, num / np.where(ok, den, 1.0), I)
    return out, ~ok


# --------------------------------------------------------------------------------------------
# Pin P1: direct double loop with the approximated kernels (same result up to rounding).
# --------------------------------------------------------------------------------------------


def bf_direct(I: np.ndarray, plan: Plan, pixels=None, window: float | None = None):
    """sum_y K~_s(y - x) K~_r(I(x) - I(y)) I(y) / sum_y K~_s(y - x) K~_r(I(x) - I(y)) with
    K~_s the lowered box kernel (eq:Box_N_terms) and K~_r the cosine series
    (eq:trigonometric_N_terms); the window is clipped to the image. `pixels` = optional list
    of (y, x) to evaluate (default: all). `window` = T restricts the range kernel to
    |I(x) - I(y)| <= T, the box B(I(x) - I(y)) of eq:trigonometric_N_terms / eq:1D_N_terms
     that the literal dimension promotion evaluates (NEXT f1).
    Returns (out, num, den) arrays / vectors."""
    I = np.asarray(I, dtype=np.float64)
    H, W = I.shape
    r = plan.radius
    Ks = spatial_kernel_values(plan.sp)
    if pixels is None:
        pixels = [(y, x) for y in range(H) for x in range(W)]
    num = np.empty(len(pixels))
    den = np.empty(len(pixels))
    for i, (y, x) in enumerate(pixels):
        ya, yb = max(0, y - r), min(H, y + r + 1)
        xa, xb = max(0, x - r), min(W, x + r + 1)
        win = I[ya:yb, xa:xb]
        ks = Ks[ya - y + r:yb - y + r, xa - x + r:xb - x + r]
        t = I[y, x] - win
        w = ks * range_kernel_approx(plan.rng, t)
        if window is not None:
            w = np.where(np.abs(t) <= window, w, 0.0)
        num[i] = np.sum(w * win)
        den[i] = np.sum(w)
    center = np.array([I[y, x] for (y, x) in pixels])
    out, _ = normalise(center, num, den)
    return out, num, den


# --------------------------------------------------------------------------------------------
# Pin P2: the paper's literal dimension-promoted 3-D box filter.
# --------------------------------------------------------------------------------------------


def bf_promoted(I_levels: np.ndarray, plan: Plan, half_window: float, n_levels: int = 256):
    """eq:numerator_2D_box_N_terms evaluated literally on integer-valued images:
    F_c(y, z) = G^c_k(y) delta_{I(y)}(z), F_s likewise; per-level 2-D box sums
    (eq:sat_sum_3D_1 via 2-D SATs); then the z-window N_{I(x)} = [I(x) - T, I(x) + T] summed
    with a 1-D SAT along z (eq:sat_sum_3D_2). Cost is n_levels times the 2-D evaluation, so this
    is for tiny images. Returns (out, num, den)."""
    I = np.asarray(I_levels)
    assert np.all(I == np.round(I)), "dimension promotion needs integer intensities (P:106)"
    Ii = I.astype(np.int64)
    If = I.astype(np.float64)
    H, W = I.shape
    num = np.zeros((H, W))
    den = np.zeros((H, W))
    # N_{I(x)} = [I(x) - T, I(x) + T] intersected with the levels [0, n_levels)
    zlo = np.clip(np.ceil(If - half_window).astype(np.int64), 0, n_levels)
    zhi = np.clip(np.floor(If + half_window).astype(np.int64), -1, n_levels - 1)
    yy, xx = np.indices((H, W))
    for k, a in zip(plan.rng.k, plan.rng.a):
        gc, gs, Gc, Gs = channels(If, k, plan.D)
        sums = []
        for X in (Gc, Gs, gc, gs):
            # I-bar(x, z): 2-D box filter of each z-slice (eq:sat_sum_3D_1)
            Ibar = np.zeros((n_levels, H, W))
            for z in range(n_levels):
                Fz = np.where(Ii == z, X, 0.0)
                if np.any(Fz != 0.0):
                    Ibar[z] = spatial_filter(Fz, plan.sp.boxes)
            # 1-D SAT along z and the window (eq:sat_sum_3D_2, eq:sat_sum_1D)
            Z = np.concatenate([np.zeros((1, H, W)), np.cumsum(Ibar, axis=0)], axis=0)
            sums.append(Z[zhi + 1, yy, xx] - Z[zlo, yy, xx])
        sGc, sGs, sgc, sgs = sums
        num += a * (gc * sGc + gs * sGs)
        den += a * (gc * sgc + gs * sgs)
    out, _ = normalise(If, num, den)
    return out, num, den


# --------------------------------------------------------------------------------------------
# Brute-force bilateral filter eq:BF, O(|N_x| |I|).
# --------------------------------------------------------------------------------------------


def spatial_kernel_exact(kind: str, sigma: float, radius: int) -> np.ndarray:
    """K_s on the square (2r+1)^2 window: Gaussian exp(-(u^2+v^2)/2 sigma^2) or box."""
    u = np.arange(-radius, radius + 1, dtype=np.float64)
    if kind == "gaussian":
        g = np.exp(-u * u / (2.0 * sigma * sigma))
        return np.outer(g, g)
    if kind == "box":
        return np.ones((2 * radius + 1, 2 * radius + 1))
    raise ValueError(kind)


def bf_bruteforce(I: np.ndarray, Ks: np.ndarray, range_fn) -> np.ndarray:
    """eq:BF with an arbitrary (2r+1)^2 spatial weight table Ks and range function K_r;
    neighbourhood clipped to the image."""
    I = np.asarray(I, dtype=np.float64)
    H, W = I.shape
    r = (Ks.shape[0] - 1) // 2
    out = np.empty_like(I)
    for y in range(H):
        ya, yb = max(0, y - r), min(H, y + r + 1)
        for x in range(W):
            xa, xb = max(0, x - r), min(W, x + r + 1)
            win = I[ya:yb, xa:xb]
            w = Ks[ya - y + r:yb - y + r, xa - x + r:xb - x + r] * range_fn(I[y, x] - win)
            out[y, x] = np.sum(w * win) / np.sum(w)
    return out


def bf_exact(I, spatial: str, sigma_s: float, radius: int, range_kind: str, sigma_r: float, **_):
    """The exact (un-approximated) BF of the configs: K_s exact on the square, K_r exact."""
    return bf_bruteforce(I, spatial_kernel_exact(spatial, sigma_s, radius), range_kernel(range_kind, sigma_r))


def psnr(a: np.ndarray, b: np.ndarray, peak: float = 255.0) -> float:
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return 120.0 if mse < 1e-12 else 10.0 * math.log10(peak * peak / mse)
