"""Every-pixel parity at the configs' full sizes: a tiled, multi-process evaluation of the oracle.

TEST INFRASTRUCTURE (imported by tests/ and tools/parity_fullsize.py only). The oracle itself
(oracle.bf.bf_box, fp64 SAT evaluation of eq:numerator_2D_box_N_terms) is called
unchanged on row bands of the image: band [a, b) is evaluated on the crop of rows
[a - r, b + r) (full width) and only rows [a, b) are kept. A kept pixel's whole window lies inside
the crop, and rows outside the image contribute nothing in both the crop and the full image
(reading Q16), so every kept value is the full-image oracle value up to fp64 rounding of the
SAT (pinned by tests/test_fullsize_harness.py against a whole-image bf_box). Bands run in
`os.cpu_count()` spawned worker processes (no CUDA in the workers).

Besides out(x) the harness returns, per pixel,
  cond(x) = den(x) / sum_b w_b |rect_b n image|   (den over the clipped spatial-kernel mass,
                                                   SURVEY 8(c) step 6)
and the oracle's fallback mask (den <= 0 or not finite, reading Q18).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor
import multiprocessing as mp

import numpy as np

MAX_ABS = 1e-3
RMSE = 1e-4


def _band_worker(args):
    crop, params, keep0, keep1 = args
    from oracle import bf, fit
    plan = fit.make_plan(**params)
    out, num, den, fb = bf.bf_box(crop, plan, return_parts=True)
    mass = bf.spatial_filter(np.ones(crop.shape), plan.sp.boxes)
    with np.errstate(divide="ignore", invalid="ignore"):
        cond = den / mass
    return out[keep0:keep1], cond[keep0:keep1].astype(np.float32), fb[keep0:keep1]


def oracle_banded(img: np.ndarray, params: dict, n_workers: int | None = None, n_bands: int | None = None,
                  pool=None):
    """(out, cond, fallback) of oracle.bf.bf_box over the whole image, evaluated band by band."""
    H, W = img.shape
    r = int(params["radius"])
    n_workers = n_workers or os.cpu_count() or 1
    n_bands = n_bands or max(1, min(H, n_workers))
    edges = [H * i // n_bands for i in range(n_bands + 1)]
    jobs = []
    for a, b in zip(edges[:-1], edges[1:]):
        if b <= a:
            continue
        ca, cb = max(0, a - r), min(H, b + r)
        jobs.append((np.ascontiguousarray(img[ca:cb]), params, a - ca, b - ca))
    out = np.empty((H, W))
    cond = np.empty((H, W), dtype=np.float32)
    fb = np.empty((H, W), dtype=bool)
    own = pool is None
    if own:
        pool = ProcessPoolExecutor(max_workers=min(n_workers, len(jobs)), mp_context=mp.get_context("spawn"))
    try:
        row = 0
        for o, c, f in pool.map(_band_worker, jobs):
            out[row:row + len(o)] = o
            cond[row:row + len(o)] = c
            fb[row:row + len(o)] = f
            row += len(o)
    finally:
        if own:
            pool.shutdown()
    assert row == H
    return out, cond, fb


def _frame_worker(args):
    img, params = args
    from oracle import bf, fit
    plan = fit.make_plan(**params)
    out, num, den, fb = bf.bf_box(img, plan, return_parts=True)
    mass = bf.spatial_filter(np.ones(img.shape), plan.sp.boxes)
    with np.errstate(divide="ignore", invalid="ignore"):
        cond = den / mass
    return out, cond.astype(np.float32), fb


def oracle_frames(frames, params: dict, n_workers: int | None = None):
    """bf_box of every frame (whole frames, one per worker task)."""
    n_workers = n_workers or os.cpu_count() or 1
    with ProcessPoolExecutor(max_workers=min(n_workers, len(frames)), mp_context=mp.get_context("spawn")) as pool:
        return list(pool.map(_frame_worker, [(f, params) for f in frames]))


def summarise(got: np.ndarray, ref: np.ndarray, cond: np.ndarray, fb_ref: np.ndarray, D: float, img: np.ndarray,
              n_worst: int = 8) -> dict:
    """Error statistics on the [0, 255] scale plus the worst and the worst-conditioned pixels."""
    got = np.asarray(got, dtype=np.float64)
    e = np.abs(got - ref) * (255.0 / D)
    finite = bool(np.all(np.isfinite(got)))
    mx = float(np.max(e)) if finite else math.inf
    rm = float(np.sqrt(np.mean(e * e))) if finite else math.inf
    H, W = got.shape
    flat_e = e.ravel()
    worst = np.argsort(flat_e)[::-1][:n_worst]
    c = np.where(np.isfinite(cond), cond, -np.inf).ravel()
    illc = np.argsort(c)[:n_worst]
    # fallback pixels of the oracle (out = I(x)); the GPU must take the same decision there
    fb_idx = np.flatnonzero(fb_ref.ravel())
    gpu_fb = got.ravel()[fb_idx] == np.asarray(img, dtype=np.float64).ravel()[fb_idx]
    return {
        "pixels": int(got.size), "max_abs": mx, "rmse": rm, "finite": finite,
        "max_abs_tol": MAX_ABS, "rmse_tol": RMSE, "pass": bool(finite and mx <= MAX_ABS and rm <= RMSE),
        "worst": [{"y": int(i // W), "x": int(i % W), "err": float(flat_e[i]), "cond": float(c[i])} for i in worst],
        "worst_conditioned": [{"y": int(i // W), "x": int(i % W), "err": float(flat_e[i]), "cond": float(c[i])}
                              for i in illc],
        "cond_min": float(np.min(c)), "n_cond_below_1e-3": int(np.sum(c < 1e-3)),
        "oracle_fallbacks": [{"y": int(i // W), "x": int(i % W), "cond": float(c[i]), "gpu_fallback": bool(g)}
                             for i, g in zip(fb_idx[:64], gpu_fb[:64])],
        "n_oracle_fallbacks": int(fb_idx.size), "n_fallback_match": int(np.sum(gpu_fb)),
    }
