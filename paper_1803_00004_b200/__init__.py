"""bf-b200: the joint-acceleration bilateral filter (arXiv 1803.00004) on the NVIDIA B200.

Thin Python layer over libbf.so (include/bf.h). PyTorch is used only for device memory and
streams; every step of the filter runs in the library's host fitter and sm_100a kernels.

    from paper_1803_00004_b200 import Plan, bilateral_filter
    plan = Plan(spatial="gaussian", range_kind="gaussian", sigma_s=16, sigma_r=0.1, radius=48,
                n_terms=16, intensity_max=1.0)
    out = bilateral_filter(plan, img_cuda_tensor)       # float32 [H, W] on the same device
"""
from __future__ import annotations

from ._bf import (BFError, Plan, apply, apply_batched, apply_host, apply_multi, config, launches, lib, version)

__all__ = ["BFError", "Plan", "apply", "apply_batched", "apply_host", "apply_multi", "bilateral_filter",
           "bilateral_filter_multi", "config", "launches", "lib", "version"]


def _check_tensor(t, plan):
    import torch
    if not t.is_cuda:
        raise ValueError("input must be a CUDA tensor (there is no CPU path)")
    want = torch.uint8 if plan.input_dtype == "u8" else torch.float32
    if t.dtype != want:
        raise TypeError(f"plan expects {want}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("input must be contiguous (row-major, pitch W)")


def bilateral_filter(plan: Plan, img, out=None, stream=None):
    """Filters a [H, W] (or [F, H, W] batch) CUDA tensor with `plan` on the current stream."""
    import torch
    _check_tensor(img, plan)
    if out is None:
        out = torch.empty(img.shape, dtype=torch.float32, device=img.device)
    s = (stream or torch.cuda.current_stream(img.device)).cuda_stream
    if img.dim() == 2:
        apply(plan, img.data_ptr(), out.data_ptr(), img.shape[0], img.shape[1], s)
    elif img.dim() == 3:
        apply_batched(plan, img.data_ptr(), out.data_ptr(), img.shape[0], img.shape[1], img.shape[2], s)
    else:
        raise ValueError("expected [H, W] or [F, H, W]")
    return out


def bilateral_filter_multi(plans, img, stream=None):
    """Filters a [H, W] CUDA tensor with up to 4 range plans that share the spatial plan, in one
    pass over shared box-filtered channels (Case 1 of P:1200-1219). Returns [len(plans), H, W]."""
    import torch
    for p in plans:
        _check_tensor(img, p)
    if img.dim() != 2:
        raise ValueError("expected [H, W]")
    out = torch.empty((len(plans),) + tuple(img.shape), dtype=torch.float32, device=img.device)
    s = (stream or torch.cuda.current_stream(img.device)).cuda_stream
    apply_multi(plans, img.data_ptr(), out.data_ptr(), img.shape[0], img.shape[1], s)
    return out
