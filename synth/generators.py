"""Synthetic images for the five BASELINE.json configs (recipe: DESIGN.md "Inputs").

Draw order is fixed so every consumer sees identical arrays for a seed:
  * ramp (configs 0, 1, 3): img[y, x] = 255*x/(W-1); then per rectangle
    x0,x1 = sorted(rng.integers(0, W, 2)), y0,y1 = sorted(rng.integers(0, H, 2)),
    v = rng.uniform(0, 255) painted over the inclusive rectangle; then
    + rng.normal(0, noise, (H, W)), clip to [0, 255], round half-to-even -> uint8.
  * sinusoid (configs 2, 4): 0.5 + sum_{i<8} (1/16) sin(2 pi f_i (cos t_i x/W + sin t_i y/H) + p_i),
    (f, t, p) drawn per sinusoid as f~U[1,64], t~U[0,2pi), p~U[0,2pi); rectangles painted with
    v~U[0,1]; + N(0, noise^2); clip to [0, 1]; float32. Config 4 multiplies by 255 (float32).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _paint_rects(img: np.ndarray, rng: np.random.Generator, n_rects: int, vmax: float) -> None:
    H, W = img.shape
    for _ in range(n_rects):
        x0, x1 = sorted(rng.integers(0, W, 2))
        y0, y1 = sorted(rng.integers(0, H, 2))
        v = rng.uniform(0.0, vmax)
        img[y0:y1 + 1, x0:x1 + 1] = v


def ramp_image(H: int, W: int, seed: int, n_rects: int, noise: float) -> np.ndarray:
    """uint8 HxW: horizontal ramp 0..255 + rectangles + Gaussian noise, clamped and rounded."""
    rng = np.random.default_rng(seed)
    x = np.arange(W, dtype=np.float64)
    img = np.broadcast_to(255.0 * x / max(W - 1, 1), (H, W)).copy()
    _paint_rects(img, rng, n_rects, 255.0)
    img = img + rng.normal(0.0, noise, (H, W))
    return np.rint(np.clip(img, 0.0, 255.0)).astype(np.uint8)


def sinusoid_image(H: int, W: int, seed: int, n_rects: int, noise: float, scale: float = 1.0) -> np.ndarray:
    """float32 HxW in [0, scale]: 8 random 2-D sinusoids + rectangles + Gaussian noise, clamped."""
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    img = np.full((H, W), 0.5)
    for _ in range(8):
        f = rng.uniform(1.0, 64.0)
        t = rng.uniform(0.0, 2.0 * np.pi)
        p = rng.uniform(0.0, 2.0 * np.pi)
        img += (1.0 / 16.0) * np.sin(2.0 * np.pi * f * (np.cos(t) * xx / W + np.sin(t) * yy / H) + p)
    _paint_rects(img, rng, n_rects, 1.0)
    img = img + rng.normal(0.0, noise, (H, W))
    img = np.clip(img, 0.0, 1.0)
    return (img * scale).astype(np.float32)


@dataclass(frozen=True)
class ConfigSpec:
    """One BASELINE.json config: image recipe + filter parameters (as given by the config text)."""
    name: str
    H: int
    W: int
    gen: str                 # "ramp" | "sinusoid"
    seeds: tuple
    n_rects: int
    noise: float
    as_f32: bool             # ramp images converted to float32 (config 1)
    scale: float             # sinusoid scale (1 or 255)
    spatial: str             # "gaussian" | "box"
    sigma_s: float
    radius: int
    range_kind: str          # "gaussian" | "tukey"
    sigma_r: float
    n_terms: int
    intensity_max: float     # D
    frames: int = 1
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "cfg0": ConfigSpec("cfg0", 256, 256, "ramp", (0,), 12, 10.0, False, 1.0,
                       "gaussian", 3.0, 9, "gaussian", 30.0, 8, 255.0),
    "cfg1": ConfigSpec("cfg1", 1024, 1024, "ramp", (1,), 64, 15.0, True, 1.0,
                       "gaussian", 8.0, 24, "gaussian", 20.0, 12, 255.0),
    "cfg2": ConfigSpec("cfg2", 4096, 4096, "sinusoid", (2,), 256, 0.04, False, 1.0,
                       "gaussian", 16.0, 48, "gaussian", 0.1, 16, 1.0),
    "cfg3": ConfigSpec("cfg3", 1080, 1920, "ramp", tuple(range(3, 67)), 128, 8.0, False, 1.0,
                       "box", 0.0, 10, "gaussian", 15.0, 10, 255.0, frames=64),
    "cfg4": ConfigSpec("cfg4", 8192, 8192, "sinusoid", (4,), 256, 0.04, False, 255.0,
                       "gaussian", 64.0, 192, "tukey", 40.0, 24, 255.0),
}


def config_input(spec: ConfigSpec, frame: int = 0, H: int | None = None, W: int | None = None) -> np.ndarray:
    """The input image of a config (optionally at a reduced HxW with the same recipe)."""
    H = spec.H if H is None else H
    W = spec.W if W is None else W
    seed = spec.seeds[frame]
    if spec.gen == "ramp":
        img = ramp_image(H, W, seed, spec.n_rects, spec.noise)
        return img.astype(np.float32) if spec.as_f32 else img
    # sinusoid recipe: noise sigma is 0.04 on the [0, 1] scale before scaling
    return sinusoid_image(H, W, seed, spec.n_rects, spec.noise, spec.scale)


def config_params(spec: ConfigSpec) -> dict:
    """Filter parameters of a config in the vocabulary of bf_plan_create."""
    return dict(spatial=spec.spatial, range_kind=spec.range_kind, sigma_s=spec.sigma_s,
                sigma_r=spec.sigma_r, radius=spec.radius, n_terms=spec.n_terms,
                intensity_max=spec.intensity_max)
