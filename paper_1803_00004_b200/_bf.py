"""ctypes binding of libbf.so (include/bf.h). Argument marshalling only: every step of the
filter runs inside the library (host fitter + sm_100a kernels). There is no CPU fallback: if
the library is missing this module raises at import."""
from __future__ import annotations

import ctypes as C
import math
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbf.so")

BF_OK, BF_ERR_INVALID_ARG, BF_ERR_UNSUPPORTED, BF_ERR_NO_MEMORY, BF_ERR_CUDA, BF_ERR_NUMERIC, BF_ERR_WORKSPACE = range(7)
KERNELS = {"auto": 0, "band": 1, "ws": 2, "ws2": 3, "ws2wide": 4}
BF_SPATIAL_GAUSSIAN, BF_SPATIAL_BOX = 0, 1
BF_RANGE_GAUSSIAN, BF_RANGE_TUKEY = 0, 1
BF_IN_U8, BF_IN_F32 = 0, 1
BF_MAX_TERMS = 32
BF_MAX_SPATIAL_TERMS = 64
BF_MAX_AXIS_BOXES = 4

SPATIAL = {"gaussian": BF_SPATIAL_GAUSSIAN, "box": BF_SPATIAL_BOX}
RANGE = {"gaussian": BF_RANGE_GAUSSIAN, "tukey": BF_RANGE_TUKEY}

#: every symbol include/bf.h declares (checked by tests/test_abi.py)
EXPORTS = ("bf_plan_options_default", "bf_plan_create", "bf_plan_destroy", "bf_plan_get_info", "bf_apply",
           "bf_apply_args_default", "bf_apply_ex", "bf_workspace_size", "bf_apply_batched", "bf_apply_config",
           "bf_apply_host", "bf_apply_launches", "bf_apply_multi", "bf_cache_size", "bf_precompute", "bf_plan_spatial_kernel", "bf_shard_frames",
           "bf_apply_cached", "bf_status_string", "bf_version")
BF_MAX_PLANS = 4


class PlanOptions(C.Structure):
    _fields_ = [("intensity_max", C.c_double), ("n_spatial_terms", C.c_int), ("input_dtype", C.c_int),
                ("m_factor", C.c_int), ("haar_levels", C.c_int), ("range_window", C.c_int)]


class LaunchConfig(C.Structure):
    _fields_ = [("n_launches", C.c_int), ("kernel", C.c_char_p), ("threads_per_cta", C.c_int), ("grid_x", C.c_int),
                ("grid_y", C.c_int), ("grid_z", C.c_int), ("tile_w", C.c_int), ("tile_h", C.c_int),
                ("smem_bytes", C.c_size_t), ("cluster_size", C.c_int), ("terms_per_cta", C.c_int),
                ("cols_per_thread", C.c_int), ("workspace_bytes", C.c_size_t),
                ("warp_map", C.c_ubyte * 24)]


class ApplyArgs(C.Structure):
    _fields_ = [("kernel", C.c_int), ("band_rows", C.c_int), ("row_begin", C.c_int), ("row_end", C.c_int),
                ("d_workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("d_fallback_count", C.c_void_p), ("d_fallback_mask", C.c_void_p), ("repair_threshold", C.c_double),
                ("d_repaired_count", C.c_void_p), ("u8_trig", C.c_int)]


class CacheDesc(C.Structure):
    _fields_ = [("k_count", C.c_int), ("H", C.c_int), ("W", C.c_int), ("input_dtype", C.c_int),
                ("intensity_max", C.c_double), ("spatial_key", C.c_ulonglong)]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_terms_eff", C.c_int), ("k", C.c_int * BF_MAX_TERMS), ("a", C.c_double * BF_MAX_TERMS),
        ("T_range", C.c_double), ("n_spatial_eff", C.c_int),
        ("sp_family", C.c_int * BF_MAX_SPATIAL_TERMS),
        ("sp_j1", C.c_int * BF_MAX_SPATIAL_TERMS), ("sp_k1", C.c_int * BF_MAX_SPATIAL_TERMS),
        ("sp_j2", C.c_int * BF_MAX_SPATIAL_TERMS), ("sp_k2", C.c_int * BF_MAX_SPATIAL_TERMS),
        ("sp_coef", C.c_double * BF_MAX_SPATIAL_TERMS),
        ("separable", C.c_int), ("nbx", C.c_int), ("nby", C.c_int),
        ("box_lo_x", C.c_int * BF_MAX_AXIS_BOXES), ("box_hi_x", C.c_int * BF_MAX_AXIS_BOXES),
        ("box_w_x", C.c_double * BF_MAX_AXIS_BOXES),
        ("box_lo_y", C.c_int * BF_MAX_AXIS_BOXES), ("box_hi_y", C.c_int * BF_MAX_AXIS_BOXES),
        ("box_w_y", C.c_double * BF_MAX_AXIS_BOXES),
        ("radius", C.c_int), ("intensity_max", C.c_double), ("input_dtype", C.c_int),
        ("spatial_rank", C.c_int), ("range_window", C.c_int), ("spatial_passes", C.c_int),
    ]


class BFError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {lib().bf_status_string(status).decode()}")


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1803_00004_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.bf_plan_options_default.argtypes = [C.POINTER(PlanOptions)]
        L.bf_plan_options_default.restype = None
        L.bf_plan_create.argtypes = [C.POINTER(P), C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                     C.POINTER(PlanOptions)]
        L.bf_plan_create.restype = C.c_int
        L.bf_plan_destroy.argtypes = [P]
        L.bf_plan_destroy.restype = C.c_int
        L.bf_plan_get_info.argtypes = [P, C.POINTER(PlanInfo)]
        L.bf_plan_get_info.restype = C.c_int
        L.bf_apply.argtypes = [P, P, P, C.c_int, C.c_int, P]
        L.bf_apply.restype = C.c_int
        L.bf_apply_batched.argtypes = [P, P, P, C.c_int, C.c_int, C.c_int, P]
        L.bf_apply_batched.restype = C.c_int
        L.bf_apply_host.argtypes = [P, P, P, C.c_int, C.c_int, P]
        L.bf_apply_host.restype = C.c_int
        L.bf_apply_multi.argtypes = [C.POINTER(P), C.c_int, P, P, C.c_int, C.c_int, P]
        L.bf_apply_multi.restype = C.c_int
        L.bf_apply_launches.argtypes = [P, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.bf_apply_launches.restype = C.c_int
        L.bf_apply_config.argtypes = [P, C.c_int, C.c_int, C.c_int, C.POINTER(ApplyArgs), C.POINTER(LaunchConfig)]
        L.bf_apply_config.restype = C.c_int
        L.bf_apply_args_default.argtypes = [C.POINTER(ApplyArgs)]
        L.bf_apply_args_default.restype = None
        L.bf_apply_ex.argtypes = [P, P, P, C.c_int, C.c_int, C.c_int, P, C.POINTER(ApplyArgs)]
        L.bf_apply_ex.restype = C.c_int
        L.bf_workspace_size.argtypes = [P, C.c_int, C.c_int, C.c_int, C.POINTER(ApplyArgs), C.POINTER(C.c_size_t)]
        L.bf_workspace_size.restype = C.c_int
        L.bf_cache_size.argtypes = [P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_size_t)]
        L.bf_cache_size.restype = C.c_int
        L.bf_precompute.argtypes = [P, C.c_int, P, C.c_int, C.c_int, P, C.c_size_t, P, C.POINTER(CacheDesc)]
        L.bf_precompute.restype = C.c_int
        L.bf_apply_cached.argtypes = [P, C.POINTER(CacheDesc), P, P, P, P, C.POINTER(ApplyArgs)]
        L.bf_apply_cached.restype = C.c_int
        L.bf_shard_frames.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.bf_shard_frames.restype = C.c_int
        L.bf_plan_spatial_kernel.argtypes = [P, C.POINTER(C.c_double), C.c_size_t]
        L.bf_plan_spatial_kernel.restype = C.c_int
        L.bf_status_string.argtypes = [C.c_int]
        L.bf_status_string.restype = C.c_char_p
        L.bf_version.argtypes = []
        L.bf_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status: int, where: str) -> None:
    if status != BF_OK:
        raise BFError(status, where)


class Plan:
    """A bf_plan (host-fitted coefficients). Mirrors bf_plan_create's arguments."""

    def __init__(self, spatial: str = "gaussian", range_kind: str = "gaussian", sigma_s: float = 3.0,
                 sigma_r: float = 30.0, radius: int = 9, n_terms: int = 8, intensity_max: float = 255.0,
                 n_spatial: int = 9, input_dtype: str = "f32", m_factor: int = 20, haar_levels: int = 4,
                 range_window: str = "full"):
        L = lib()
        opt = PlanOptions()
        L.bf_plan_options_default(C.byref(opt))
        opt.intensity_max = float(intensity_max)
        opt.n_spatial_terms = int(n_spatial)
        opt.input_dtype = BF_IN_U8 if input_dtype in ("u8", "uint8") else BF_IN_F32
        opt.m_factor = int(m_factor)
        opt.haar_levels = int(haar_levels)
        opt.range_window = {"full": 0, "literal": 1}[range_window]
        h = C.c_void_p()
        st = L.bf_plan_create(C.byref(h), SPATIAL[spatial], RANGE[range_kind], float(sigma_s), float(sigma_r),
                              int(radius), int(n_terms), C.byref(opt))
        _check(st, "bf_plan_create")
        self._h = h
        self.input_dtype = "u8" if opt.input_dtype == BF_IN_U8 else "f32"

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def info(self) -> dict:
        inf = PlanInfo()
        _check(lib().bf_plan_get_info(self._h, C.byref(inf)), "bf_plan_get_info")
        n, ns = inf.n_terms_eff, inf.n_spatial_eff
        return dict(
            k=list(inf.k[:n]), a=list(inf.a[:n]), T_range=inf.T_range,
            spatial_terms=[(inf.sp_family[i], inf.sp_j1[i], inf.sp_k1[i], inf.sp_j2[i], inf.sp_k2[i], inf.sp_coef[i])
                           for i in range(ns)],
            separable=bool(inf.separable),
            boxes_x=[(inf.box_lo_x[i], inf.box_hi_x[i], inf.box_w_x[i]) for i in range(inf.nbx)],
            boxes_y=[(inf.box_lo_y[i], inf.box_hi_y[i], inf.box_w_y[i]) for i in range(inf.nby)],
            radius=inf.radius, intensity_max=inf.intensity_max, spatial_rank=inf.spatial_rank, spatial_passes=inf.spatial_passes,
            range_window="literal" if inf.range_window == 1 else "full",
            input_dtype="u8" if inf.input_dtype == BF_IN_U8 else "f32")

    def spatial_kernel(self):
        """K~_s(v, u) on the (2r+1)^2 integer offsets as the GPU path applies it (numpy [v+r, u+r])."""
        import numpy as np
        r = self.info()["radius"]
        n = 2 * r + 1
        K = np.zeros((n, n), dtype=np.float64)
        _check(lib().bf_plan_spatial_kernel(self._h, K.ctypes.data_as(C.POINTER(C.c_double)), K.size),
               "bf_plan_spatial_kernel")
        return K

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().bf_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


def make_args(kernel: str = "auto", band_rows: int = 0, rows=None, workspace=(0, 0), fallback_count: int = 0,
              fallback_mask: int = 0, repair_threshold: float = 0.0, u8_trig: str = "lut",
              repaired_count: int = 0) -> ApplyArgs:
    """bf_apply_args: kernel choice, band height, output row range, workspace (ptr, bytes), device
    fallback counter / mask pointers (0 = off), fp64 repair threshold (0 = default, < 0 = off)."""
    a = ApplyArgs()
    lib().bf_apply_args_default(C.byref(a))
    a.kernel = KERNELS[kernel]
    a.band_rows = int(band_rows)
    if rows is not None:
        a.row_begin, a.row_end = int(rows[0]), int(rows[1])
    a.d_workspace = C.c_void_p(int(workspace[0])) if workspace[0] else None
    a.workspace_bytes = int(workspace[1])
    a.d_fallback_count = C.c_void_p(int(fallback_count)) if fallback_count else None
    a.d_fallback_mask = C.c_void_p(int(fallback_mask)) if fallback_mask else None
    a.repair_threshold = float(repair_threshold)
    a.u8_trig = {"lut": 0, "direct": 1}[u8_trig]
    a.d_repaired_count = C.c_void_p(int(repaired_count)) if repaired_count else None
    return a


def apply(plan: Plan, d_in: int, d_out: int, H: int, W: int, stream: int = 0) -> None:
    """bf_apply on raw device pointers (ints) and a raw cudaStream_t (int)."""
    _check(lib().bf_apply(plan.handle, C.c_void_p(d_in), C.c_void_p(d_out), int(H), int(W), C.c_void_p(stream)),
           "bf_apply")


def apply_ex(plan: Plan, d_in: int, d_out: int, n_frames: int, H: int, W: int, stream: int = 0,
             args: ApplyArgs | None = None) -> None:
    """bf_apply_ex (optional arguments: see make_args)."""
    _check(lib().bf_apply_ex(plan.handle, C.c_void_p(d_in), C.c_void_p(d_out), int(n_frames), int(H), int(W),
                             C.c_void_p(stream), C.byref(args) if args is not None else None), "bf_apply_ex")


def workspace_size(plan: Plan, H: int, W: int, n_frames: int = 1, args: ApplyArgs | None = None) -> int:
    n = C.c_size_t(0)
    _check(lib().bf_workspace_size(plan.handle, int(n_frames), int(H), int(W),
                                   C.byref(args) if args is not None else None, C.byref(n)), "bf_workspace_size")
    return n.value


def cache_size(plan: Plan, k_count: int, H: int, W: int) -> int:
    n = C.c_size_t(0)
    _check(lib().bf_cache_size(plan.handle, int(k_count), int(H), int(W), C.byref(n)), "bf_cache_size")
    return n.value


def precompute(plan: Plan, k_count: int, d_in: int, H: int, W: int, d_cache: int, cache_bytes: int,
               stream: int = 0) -> CacheDesc:
    """bf_precompute (Case 1, phase 1): box-filtered channels of k = 0 .. k_count-1 into d_cache."""
    d = CacheDesc()
    _check(lib().bf_precompute(plan.handle, int(k_count), C.c_void_p(d_in), int(H), int(W), C.c_void_p(d_cache),
                               int(cache_bytes), C.c_void_p(stream), C.byref(d)), "bf_precompute")
    return d


def apply_cached(plan: Plan, desc: CacheDesc, d_cache: int, d_in: int, d_out: int, stream: int = 0,
                 args: ApplyArgs | None = None) -> None:
    """bf_apply_cached (Case 1, phase 2): combine-only pass of a range plan over the cache."""
    _check(lib().bf_apply_cached(plan.handle, C.byref(desc), C.c_void_p(d_cache), C.c_void_p(d_in),
                                 C.c_void_p(d_out), C.c_void_p(stream), C.byref(args) if args is not None else None),
           "bf_apply_cached")


def apply_batched(plan: Plan, d_in: int, d_out: int, n_frames: int, H: int, W: int, stream: int = 0) -> None:
    _check(lib().bf_apply_batched(plan.handle, C.c_void_p(d_in), C.c_void_p(d_out), int(n_frames), int(H), int(W),
                                  C.c_void_p(stream)), "bf_apply_batched")


def apply_host(plan: Plan, h_in: int, h_out: int, H: int, W: int, stream: int = 0) -> None:
    """bf_apply_host on raw host pointers (copies in, filters, copies out, synchronises)."""
    _check(lib().bf_apply_host(plan.handle, C.c_void_p(h_in), C.c_void_p(h_out), int(H), int(W), C.c_void_p(stream)),
           "bf_apply_host")


def apply_multi(plans, d_in: int, d_out: int, H: int, W: int, stream: int = 0) -> None:
    """bf_apply_multi: several range plans over one pass of shared box-filtered channels (Case 1);
    d_out holds len(plans) H x W float32 images back to back."""
    arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
    _check(lib().bf_apply_multi(arr, len(plans), C.c_void_p(d_in), C.c_void_p(d_out), int(H), int(W),
                                C.c_void_p(stream)), "bf_apply_multi")


def launches(plan: Plan, H: int, W: int) -> int:
    """Kernel launches one bf_apply of an H x W image enqueues (bf_apply_launches)."""
    n = C.c_int(0)
    _check(lib().bf_apply_launches(plan.handle, int(H), int(W), C.byref(n)), "bf_apply_launches")
    return n.value


def config(plan: Plan, H: int, W: int, n_frames: int = 1, args: ApplyArgs | None = None) -> dict:
    """Launch configuration of bf_apply(_ex) for this shape (bf_apply_config): kernel name,
    threads per CTA, grid, output tile, dynamic shared memory, launches, cluster size, terms per
    CTA, columns per vertical-pass thread, workspace bytes."""
    c = LaunchConfig()
    _check(lib().bf_apply_config(plan.handle, int(n_frames), int(H), int(W),
                                 C.byref(args) if args is not None else None, C.byref(c)), "bf_apply_config")
    return {"kernel": c.kernel.decode(), "launches": c.n_launches, "threads_per_cta": c.threads_per_cta,
            "grid": (c.grid_x, c.grid_y, c.grid_z), "tile": (c.tile_w, c.tile_h), "smem_bytes": c.smem_bytes,
            "cluster": c.cluster_size, "terms_per_cta": c.terms_per_cta, "cols_per_thread": c.cols_per_thread,
            "workspace_bytes": c.workspace_bytes, "warp_map": list(c.warp_map)}


def shard_frames(n_frames: int, n_parts: int, part: int) -> tuple:
    """(first, count): the contiguous block of frames part `part` of n_parts filters (bf_shard_frames)."""
    f, c = C.c_int(), C.c_int()
    _check(lib().bf_shard_frames(int(n_frames), int(n_parts), int(part), C.byref(f), C.byref(c)), "bf_shard_frames")
    return f.value, c.value


def version() -> str:
    return lib().bf_version().decode()


def is_inf(x: float) -> bool:
    return math.isinf(x)
