"""bf-b200: the joint-acceleration bilateral filter (arXiv 1803.00004) on the NVIDIA B200.

Thin Python layer over libbf.so (include/bf.h). PyTorch is used only for device memory and
streams; every step of the filter runs in the library's host fitter and sm_100a kernels.

    from paper_1803_00004_b200 import Plan, bilateral_filter
    plan = Plan(spatial="gaussian", range_kind="gaussian", sigma_s=16, sigma_r=0.1, radius=48,
                n_terms=16, intensity_max=1.0)
    out = bilateral_filter(plan, img_cuda_tensor)       # float32 [H, W] on the same device
"""
from __future__ import annotations

from ._bf import (BFError, CacheDesc, Plan, apply, apply_batched, apply_cached, apply_ex, apply_host, apply_multi,
                  cache_size, config, launches, lib, make_args, precompute, shard_frames, version, workspace_size)

__all__ = ["BFError", "CacheDesc", "Plan", "apply", "apply_batched", "apply_cached", "apply_ex", "apply_host",
           "apply_multi", "bilateral_filter", "bilateral_filter_multi", "cache_size", "config", "launches", "lib",
           "make_args", "precompute", "shard_frames", "version", "workspace_size", "RangeCache"]


def _check_tensor(t, plan):
    import torch
    if not t.is_cuda:
        raise ValueError("input must be a CUDA tensor (there is no CPU path)")
    want = torch.uint8 if plan.input_dtype == "u8" else torch.float32
    if t.dtype != want:
        raise TypeError(f"plan expects {want}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("input must be contiguous (row-major, pitch W)")


def bilateral_filter(plan: Plan, img, out=None, stream=None, kernel: str = "auto", band_rows: int = 0,
                     fallback_count=None, fallback_mask=None, repair_threshold: float = 0.0, u8_trig: str = "lut",
                     repaired_count=None):
    """Filters a [H, W] (or [F, H, W] batch) CUDA tensor with `plan` on the current stream.

    Multi-pass plans get a workspace from torch's allocator (the caller's memory: the library
    itself never allocates). fallback_count: optional int64 CUDA tensor [1] incremented by the
    number of pixels whose denominator was <= 0 (out = I(x)); fallback_mask: optional uint8 CUDA
    tensor shaped like img (1 there, else 0). repair_threshold: see bf_apply_args (0 = default,
    < 0 = no fp64 repair of ill-conditioned pixels)."""
    import torch
    _check_tensor(img, plan)
    if img.dim() not in (2, 3):
        raise ValueError("expected [H, W] or [F, H, W]")
    if out is None:
        out = torch.empty(img.shape, dtype=torch.float32, device=img.device)
    s = (stream or torch.cuda.current_stream(img.device)).cuda_stream
    F, H, W = (1,) + tuple(img.shape) if img.dim() == 2 else tuple(img.shape)
    args = make_args(kernel=kernel, band_rows=band_rows,
                     fallback_count=fallback_count.data_ptr() if fallback_count is not None else 0,
                     fallback_mask=fallback_mask.data_ptr() if fallback_mask is not None else 0,
                     repair_threshold=repair_threshold, u8_trig=u8_trig,
                     repaired_count=repaired_count.data_ptr() if repaired_count is not None else 0)
    ws = workspace_size(plan, H, W, F, args)
    wst = None
    if ws:
        wst = torch.empty(ws, dtype=torch.uint8, device=img.device)
        args.d_workspace = wst.data_ptr()
        args.workspace_bytes = ws
    apply_ex(plan, img.data_ptr(), out.data_ptr(), F, H, W, s, args)
    if wst is not None:
        wst.record_stream(stream or torch.cuda.current_stream(img.device))
    return out


class RangeCache:
    """Case 1 of the paper's pre-computation on a [H, W] CUDA tensor: the box-filtered
    channels of k = 0 .. k_count-1 are computed once (bf_precompute); any range plan sharing the
    spatial plan is then applied by a combine-only pass (bf_apply_cached), bitwise equal to
    bilateral_filter. The cache is a torch CUDA tensor (4 * k_count * H * W int32)."""

    def __init__(self, plan: Plan, img, k_count: int, stream=None):
        import torch
        _check_tensor(img, plan)
        if img.dim() != 2:
            raise ValueError("expected [H, W]")
        self.img = img
        H, W = img.shape
        n = cache_size(plan, k_count, H, W)
        self.buf = torch.empty(n, dtype=torch.uint8, device=img.device)
        s = (stream or torch.cuda.current_stream(img.device)).cuda_stream
        self.desc = precompute(plan, k_count, img.data_ptr(), H, W, self.buf.data_ptr(), n, s)

    def apply(self, plan: Plan, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.img.shape, dtype=torch.float32, device=self.img.device)
        s = (stream or torch.cuda.current_stream(self.img.device)).cuda_stream
        apply_cached(plan, self.desc, self.buf.data_ptr(), self.img.data_ptr(), out.data_ptr(), s)
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
