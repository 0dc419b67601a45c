"""The C-ABI library: loads, exports every symbol include/bf.h declares, validates arguments,
and its host fitter agrees with the independent oracle fitter. No GPU compute calls."""
import math
import os
import re

import numpy as np
import pytest

from oracle import fit
from synth import CONFIGS, config_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bfmod():
    from paper_1803_00004_b200 import build
    build.build()
    import paper_1803_00004_b200._bf as b
    return b


def header_functions():
    src = open(os.path.join(ROOT, "include", "bf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*BF_API\s+(?:const\s+)?[a-z_]+\**\s+\**(bf_[a-z_]+)\s*\(", src, flags=re.M)))


def test_header_declares_expected_api():
    assert header_functions() == sorted(["bf_plan_options_default", "bf_plan_create", "bf_plan_destroy",
                                         "bf_plan_get_info", "bf_apply", "bf_apply_args_default", "bf_apply_ex",
                                         "bf_workspace_size", "bf_apply_batched", "bf_apply_host",
                                         "bf_apply_config", "bf_apply_launches", "bf_apply_multi",
                                         "bf_cache_size", "bf_precompute", "bf_apply_cached",
                                         "bf_plan_spatial_kernel", "bf_shard_frames", "bf_status_string", "bf_version"])


def test_library_exports_every_declared_symbol(bfmod):
    L = bfmod.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    assert sorted(bfmod.EXPORTS) == header_functions()
    out = os.popen(f"nm -D --defined-only {bfmod.LIB_PATH}").read()
    exported = set(re.findall(r" T (bf_\w+)", out))
    assert exported == set(header_functions())          # nothing else leaks out of the ABI


def test_status_strings_and_version(bfmod):
    L = bfmod.lib()
    for s in range(7):
        assert L.bf_status_string(s).decode().startswith("BF_")
    assert bfmod.version().startswith("bf-b200")


def test_invalid_arguments_rejected(bfmod):
    import ctypes as C
    L = bfmod.lib()
    h = C.c_void_p(123)
    assert L.bf_plan_create(C.byref(h), 0, 0, 3.0, 30.0, 9, 0, None) == bfmod.BF_ERR_INVALID_ARG
    assert h.value is None                                   # *out = NULL on failure
    assert L.bf_plan_create(C.byref(h), 0, 0, -1.0, 30.0, 9, 8, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_plan_create(C.byref(h), 0, 0, 3.0, 0.0, 9, 8, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_plan_create(C.byref(h), 0, 0, 3.0, 30.0, -1, 8, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_plan_create(C.byref(h), 7, 0, 3.0, 30.0, 9, 8, None) == bfmod.BF_ERR_UNSUPPORTED
    assert L.bf_plan_create(C.byref(h), 0, 9, 3.0, 30.0, 9, 8, None) == bfmod.BF_ERR_UNSUPPORTED
    assert L.bf_plan_create(None, 0, 0, 3.0, 30.0, 9, 8, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_plan_create(C.byref(h), 0, 0, 3.0, 30.0, 9, 33, None) == bfmod.BF_ERR_INVALID_ARG
    p = bfmod.Plan()
    # argument validation of bf_apply happens before any CUDA call
    assert L.bf_apply(p.handle, None, C.c_void_p(16), 4, 4, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_apply(p.handle, C.c_void_p(16), C.c_void_p(32), 0, 4, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_apply(p.handle, C.c_void_p(16), C.c_void_p(16), 4, 4, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_apply(None, C.c_void_p(16), C.c_void_p(32), 4, 4, None) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_plan_destroy(None) == bfmod.BF_OK


def _oracle_key_to_c(h):
    return (-1, 0) if h == fit.PHI else (h[1], h[2])


@pytest.mark.parametrize("cfg", sorted(CONFIGS))
@pytest.mark.parametrize("n_spatial", [9, 5, 1])
def test_plan_matches_oracle(bfmod, cfg, n_spatial):
    """Cross-check of two independent fitters: same k set, a_k within 1e-12 relative, same
    selected Haar terms and coefficients, and the GPU's separable factors reproduce the
    oracle's lowered box kernel K~_s at every integer offset."""
    p = config_params(CONFIGS[cfg])
    op = fit.make_plan(**p, n_spatial=n_spatial)
    gp = bfmod.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                    radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                    n_spatial=n_spatial)
    info = gp.info()
    assert info["k"] == op.rng.k
    amax = max(abs(x) for x in op.rng.a)
    assert np.max(np.abs(np.array(info["a"]) - np.array(op.rng.a))) <= 1e-12 * amax
    assert len(info["spatial_terms"]) == len(op.sp.terms)
    for (fam, j1, k1, j2, k2, c), (a, b, oc) in zip(info["spatial_terms"], op.sp.terms):
        assert fam == fit.family(a, b)
        assert (j1, k1) == _oracle_key_to_c(a) and (j2, k2) == _oracle_key_to_c(b)
        assert abs(c - oc) <= 1e-12 * max(abs(oc), 1e-300)
    Ko = fit.spatial_kernel_values(op.sp)
    r = p["radius"]
    if info["separable"]:
        fx = np.zeros(2 * r + 1)
        fy = np.zeros(2 * r + 1)
        for lo, hi, w in info["boxes_x"]:
            fx[lo + r:hi + r + 1] += w
        for lo, hi, w in info["boxes_y"]:
            fy[lo + r:hi + r + 1] += w
        Kg = np.outer(fy, fx)
        assert np.max(np.abs(Kg - Ko)) <= 1e-12 * np.max(np.abs(Ko))
    else:
        assert n_spatial == 5       # the paper's 3-box plan f1+f2+f3 is rank 2 (NEXT f3)


def test_plan_edge_parameters(bfmod):
    inf = bfmod.Plan(sigma_r=math.inf, n_terms=6).info()
    assert inf["k"] == [0] and abs(inf["a"][0] - 1.0) < 1e-12          # K_r == 1: DC only (N_eff < N)
    r0 = bfmod.Plan(radius=0).info()
    assert r0["boxes_x"] == [(0, 0, r0["boxes_x"][0][2])] and r0["separable"]
    box = bfmod.Plan(spatial="box", radius=10).info()
    assert len(box["spatial_terms"]) == 1 and box["boxes_x"][0][:2] == (-10, 10)


def test_launch_count_query(bfmod):
    """bf_apply_launches: one launch for every BASELINE config (cfg4's 24 terms at r = 192 split
    over a 3-CTA cluster instead of two workspace passes), argument validation; host-only."""
    import ctypes as C
    L = bfmod.lib()
    for cfg, want in (("cfg0", 1), ("cfg2", 1), ("cfg3", 1), ("cfg4", 1)):
        p = config_params(CONFIGS[cfg])
        plan = bfmod.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"],
                          sigma_r=p["sigma_r"], radius=p["radius"], n_terms=p["n_terms"],
                          intensity_max=p["intensity_max"])
        assert bfmod.launches(plan, 64, 64) == want, cfg
    n = C.c_int(7)
    assert L.bf_apply_launches(None, 4, 4, C.byref(n)) == bfmod.BF_ERR_INVALID_ARG
    assert L.bf_apply_launches(plan.handle, 0, 4, C.byref(n)) == bfmod.BF_ERR_INVALID_ARG


def test_launch_config_query(bfmod):
    """bf_apply_config describes the launches without device work: kernel 2b (768 threads) for the
    separable N_s = 9 plans, one column per vertical-pass thread and one CTA per strip while the
    halo leaves a strip >= 256 wide (cfg0-cfg3); cfg4's r = 192 halo takes two columns per thread
    (768 extended columns) and its 24 terms split over a cluster of 3 CTAs (8 terms each), one
    launch and no workspace. The kernel argument forces kernels 1 / 2 (one pass per 8 or 16
    terms, with a workspace); the literal kernel for range_window='literal'; the grid covers the
    image."""
    import ctypes as C
    for cfg, cols, cluster in (("cfg2", 1, 1), ("cfg1", 1, 1), ("cfg0", 1, 1), ("cfg3", 1, 1), ("cfg4", 2, 3)):
        spec = CONFIGS[cfg]
        p = config_params(spec)
        u8 = spec.gen == "ramp" and not spec.as_f32
        plan = bfmod.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"],
                          sigma_r=p["sigma_r"], radius=p["radius"], n_terms=p["n_terms"],
                          intensity_max=p["intensity_max"], input_dtype="u8" if u8 else "f32")
        c = bfmod.config(plan, spec.H, spec.W)
        assert c["kernel"] == "bf_ws2_kernel" and c["launches"] == 1 == bfmod.launches(plan, spec.H, spec.W), cfg
        assert (c["cols_per_thread"], c["cluster"], c["workspace_bytes"]) == (cols, cluster, 0), (cfg, c)
        tw, th = c["tile"]
        gx, gy, gz = c["grid"]
        strips = gx // cluster
        assert gx % cluster == 0 and strips * tw >= spec.W > (strips - 1) * tw and gy * th >= spec.H > (gy - 1) * th
        assert gz == 1 and c["smem_bytes"] <= 227 * 1024 and c["threads_per_cta"] == 768
        halo = 2 * p["radius"]
        widest = min(320 if cols == 1 else 352, 384 * cols - halo)
        assert tw == widest or (tw % 32 == 0 and 128 <= tw < widest), (cfg, tw)
        if cluster > 1:
            assert c["terms_per_cta"] * cluster >= len(plan.info()["k"]) > c["terms_per_cta"] * (cluster - 1)
        # warp roles: a permutation of the 24 logical warps. The WORKING warps of each role (FH: one
        # per 32 output columns, S: one per 32-channel group, V: one per 32 extended columns) are
        # placed over the four SM sub-partitions (physical warp mod 4) by the rule the on-GPU search
        # found (bf_apply.cu, ws2_warp_map): the S warps share one sub-partition, the FH warps are
        # spread evenly over the other three, the V warps evenly over all four
        m = c["warp_map"]
        assert sorted(m) == list(range(24)), (cfg, m)
        nfh, ns = (10, 2) if cols == 1 else (11, 1)
        nk = min(c["terms_per_cta"], len(plan.info()["k"]))
        wv = (tw + halo + 7) // 8 * 8
        ngrp = (4 * nk + 31) // 32
        fq, sq, vq = [0] * 4, [0] * 4, [0] * 4
        for pw, l in enumerate(m):
            if l < nfh:
                fq[pw % 4] += 32 * l < tw
            elif l < nfh + ns:
                sq[pw % 4] += l - nfh < ngrp
            else:
                vq[pw % 4] += 32 * (l - nfh - ns) < wv
        assert sorted(sq) == [0, 0, 0, min(ns, ngrp)], (cfg, sq)
        others = [fq[q] for q in range(4) if sq[q] == 0]
        assert max(others) - min(others) <= 1 and max(vq) - min(vq) <= 1, (cfg, fq, vq)
    spec = CONFIGS["cfg2"]
    p = config_params(spec)
    plan = bfmod.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                      radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"])
    for k, name, threads in (("band", "bf_band_kernel", 256), ("ws", "bf_ws_kernel", 640)):
        c = bfmod.config(plan, 333, 361, args=bfmod.make_args(kernel=k))
        assert (c["kernel"], c["threads_per_cta"], c["tile"][0]) == (name, threads, 256 - 2 * p["radius"])
    # cfg4 on kernel 1 (forced): two passes of 16 terms through a workspace of 16 B per pixel
    p4 = config_params(CONFIGS["cfg4"])
    plan4 = bfmod.Plan(spatial=p4["spatial"], range_kind=p4["range_kind"], sigma_s=p4["sigma_s"],
                       sigma_r=p4["sigma_r"], radius=p4["radius"], n_terms=p4["n_terms"],
                       intensity_max=p4["intensity_max"])
    c = bfmod.config(plan4, 1000, 900, args=bfmod.make_args(kernel="band"))
    assert c["kernel"] == "bf_band_kernel" and c["launches"] == 2 and c["workspace_bytes"] == 16 * 1000 * 900
    assert bfmod.workspace_size(plan4, 1000, 900, args=bfmod.make_args(kernel="band")) == 16 * 1000 * 900
    assert bfmod.workspace_size(plan4, 1000, 900) == 0
    c = bfmod.config(plan, 100, 100, args=bfmod.make_args(band_rows=7))
    assert c["tile"][1] == 7 and c["grid"][1] == 15
    lit = bfmod.Plan(range_window="literal", input_dtype="u8", radius=10, n_terms=4)
    assert bfmod.config(lit, 100, 100)["kernel"] == "bf_literal_kernel"
    c = bfmod.LaunchConfig()
    assert bfmod.lib().bf_apply_config(None, 1, 4, 4, None, C.byref(c)) == bfmod.BF_ERR_INVALID_ARG
    assert bfmod.lib().bf_apply_config(plan.handle, 0, 4, 4, None, C.byref(c)) == bfmod.BF_ERR_INVALID_ARG


def test_multi_pass_plan_needs_workspace(bfmod):
    """bf_apply never allocates: a plan that runs in several passes (here a forced kernel 1 on a
    24-term plan, or a rank-2 N_s = 5 plan with 12 terms) returns BF_ERR_WORKSPACE without a
    workspace, before any device work."""
    import ctypes as C
    L = bfmod.lib()
    p = config_params(CONFIGS["cfg1"])
    plan = bfmod.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                      radius=p["radius"], n_terms=p["n_terms"], n_spatial=5)
    assert bfmod.config(plan, 64, 64)["launches"] == 2
    assert L.bf_apply(plan.handle, C.c_void_p(16), C.c_void_p(4096), 64, 64, None) == bfmod.BF_ERR_WORKSPACE
    a = bfmod.make_args(workspace=(8192, 100))
    assert L.bf_apply_ex(plan.handle, C.c_void_p(16), C.c_void_p(4096), 1, 64, 64, None, C.byref(a)) == \
        bfmod.BF_ERR_WORKSPACE


def test_multi_plan_validation(bfmod):
    """bf_apply_multi takes separable plans with at most two boxes per axis (N_s = 2 /
    5 plans were silently wrong or failed late): others are BF_ERR_UNSUPPORTED before any device
    work, and so is a union of more than 16 terms."""
    import ctypes as C
    L = bfmod.lib()
    for ns in (5, 25):
        a = bfmod.Plan(sigma_s=4.0, radius=12, n_terms=4, n_spatial=ns)
        b = bfmod.Plan(sigma_s=4.0, radius=12, n_terms=4, n_spatial=ns, sigma_r=20.0)
        arr = (C.c_void_p * 2)(a.handle.value, b.handle.value)
        assert L.bf_apply_multi(arr, 2, C.c_void_p(16), C.c_void_p(4096), 32, 32, None) == bfmod.BF_ERR_UNSUPPORTED
    a = bfmod.Plan(n_terms=12, sigma_r=10.0)
    b = bfmod.Plan(n_terms=20, sigma_r=10.0)
    assert len(set(a.info()["k"]) | set(b.info()["k"])) > 16
    arr = (C.c_void_p * 2)(a.handle.value, b.handle.value)
    assert L.bf_apply_multi(arr, 2, C.c_void_p(16), C.c_void_p(4096), 32, 32, None) == bfmod.BF_ERR_UNSUPPORTED


def test_spatial_rank_of_the_gpu_form(bfmod):
    """bf_plan_info.spatial_rank: 1 for the separable default plans (N_s = 9, box K_s), 2 for the
    paper's three-box plan (N_s = 5); the rank-2 form's terms reproduce the lowered kernel."""
    p = config_params(CONFIGS["cfg1"])
    for ns, want in ((9, 1), (5, 2), (1, 1)):
        plan = bfmod.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"],
                          sigma_r=p["sigma_r"], radius=p["radius"], n_terms=p["n_terms"], n_spatial=ns)
        assert plan.info()["spatial_rank"] == want, ns
    box = bfmod.Plan(spatial="box", range_kind="gaussian", sigma_s=1.0, sigma_r=15.0, radius=10, n_terms=4)
    assert box.info()["spatial_rank"] == 1


@pytest.mark.parametrize("cfg,over", [("cfg0", {}), ("cfg3", {}), ("cfg0", {"range_kind": "tukey", "sigma_r": 40.0})])
def test_literal_plan_matches_oracle(bfmod, cfg, over):
    """range_window='literal' (NEXT f1): T_range = T_r = K_r^{-1}(0.01) and the range fit on
    [-T_r, T_r] agree with the oracle's independent literal fit."""
    p = dict(config_params(CONFIGS[cfg]))
    p.update(over)
    op = fit.make_literal_plan(**p)
    gp = bfmod.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                    radius=p["radius"], n_terms=p["n_terms"], input_dtype="u8", range_window="literal")
    info = gp.info()
    assert info["range_window"] == "literal"
    assert abs(info["T_range"] - fit.truncation_radius(p["range_kind"], p["sigma_r"])) <= 1e-12 * info["T_range"]
    assert info["k"] == op.rng.k
    amax = max(abs(x) for x in op.rng.a)
    assert np.max(np.abs(np.array(info["a"]) - np.array(op.rng.a))) <= 1e-12 * amax


@pytest.mark.parametrize("n_spatial,levels,radius", [(13, 4, 9), (16, 4, 24), (17, 4, 48), (25, 4, 9), (25, 2, 24),
                                                     (36, 4, 48), (49, 4, 9), (64, 2, 9), (5, 4, 192), (9, 4, 48)])
def test_spatial_kernel_factorisation_matches_oracle_lowering(bfmod, n_spatial, levels, radius):
    """NEXT f3: every spatial plan the GPU path runs is a sum of separable
    box products (one for N_s = 9, the rank-2 box-pair form for N_s = 5, otherwise the exact rank-R
    passes of bf_plan.cpp: general_passes). Their sum must equal the oracle's independent Appendix-A
    lowering (oracle.fit.spatial_kernel_values of the boxes of eq:2D_box_N_terms) on every offset."""
    sigma = radius / 3.0
    plan = bfmod.Plan(spatial="gaussian", range_kind="gaussian", sigma_s=sigma, sigma_r=20.0, radius=radius,
                      n_terms=4, n_spatial=n_spatial, haar_levels=levels)
    info = plan.info()
    K = plan.spatial_kernel()
    ref = fit.spatial_kernel_values(fit.fit_spatial("gaussian", sigma, radius, n_spatial, levels))
    assert np.max(np.abs(K - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert info["spatial_passes"] >= 1 and info["spatial_rank"] >= 1
    if n_spatial == 9 or (n_spatial in (25, 64) and levels == 2):
        assert info["spatial_rank"] == 1                 # separable (Form 2 / Form 4)
    if n_spatial not in (5, 9) and levels == 4:
        assert info["spatial_rank"] == np.linalg.matrix_rank(ref, tol=1e-10 * np.max(np.abs(ref)))
