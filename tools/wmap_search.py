"""Empirical search over kernel 2b's warp-role maps (physical warp -> logical warp) on the GPU.

Needs a search build of the library (the map read from the environment):
    python tools/build_variant.py wenv "-DBF_WMAP_ENV=1" bf_apply.cu
    python tools/wmap_search.py cfg2,cfg3 [max_candidates] > gpurun_out/wmap_search.txt

A candidate is a count layout: how many WORKING warps of each role (FH, S, V with two / one
columns) every SM sub-partition (physical warp id mod 4) runs; idle warps fill the rest. Layouts
are enumerated up to the symmetry of the sub-partitions, timed (CUDA events, L2 flushed, median),
and the best ones re-timed with several orders of the roles inside a sub-partition."""
import itertools
import json
import os
import random
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1803_00004_b200._bf as b  # noqa: E402

b.LIB_PATH = os.path.join(ROOT, "tools", "var", "libbf_wenv.so")
from synth import CONFIGS, config_input, config_params  # noqa: E402


def compositions(n, parts, cap):
    if parts == 1:
        if n <= cap:
            yield (n,)
        return
    for i in range(min(n, cap) + 1):
        for rest in compositions(n - i, parts - 1, cap):
            yield (i,) + rest


def layouts(counts):
    """All distributions of the working warps (one count per class) over four sub-partitions of
    six warps, up to permutation of the sub-partitions."""
    seen = set()
    per_class = [list(compositions(c, 4, 6)) for c in counts]
    for combo in itertools.product(*per_class):
        sub = tuple(sorted(tuple(cl[q] for cl in combo) for q in range(4)))
        if any(sum(t) > 6 for t in sub) or sub in seen:
            continue
        seen.add(sub)
        yield sub


def build_map(sub, classes, idle, order, idle_at=None):
    """sub: per sub-partition the counts per class; classes: logical warps of each class (working);
    idle: idle logical warps; order: class order inside a sub-partition; idle_at: position of the
    idle warps in a sub-partition's slot sequence (None = last)."""
    pools = [list(c) for c in classes]
    idle = list(idle)
    m = [0] * 24
    for q in range(4):
        seq = []
        for ci in order:
            for _ in range(sub[q][ci]):
                seq.append(pools[ci].pop(0))
        while len(seq) < 6:
            if idle_at is None:
                seq.append(idle.pop(0))
            else:
                seq.insert(min(idle_at, len(seq)), idle.pop(0))
        for i, l in enumerate(seq):
            m[q + 4 * i] = l
    return m


def main():
    cfgs = sys.argv[1].split(",")
    maxc = int(sys.argv[2]) if len(sys.argv) > 2 else 1200
    random.seed(0)
    for cfg in cfgs:
        spec = CONFIGS[cfg]
        p = config_params(spec)
        img = config_input(spec)
        if img.ndim == 3:
            img = img[0]
        u8 = img.dtype.name == "uint8"
        plan = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                      radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                      input_dtype="u8" if u8 else "f32")
        H, W = img.shape
        os.environ.pop("BF_WMAP_OVERRIDE", None)
        c = b.config(plan, H, W)
        cols, tw = c["cols_per_thread"], c["tile"][0]
        nfh, ns = (10, 2) if cols == 1 else (11, 1)
        wv = (tw + 2 * p["radius"] + 7) // 8 * 8
        nkc = min(c["terms_per_cta"], len(plan.info()["k"]))
        ngrp = (4 * nkc + 31) // 32
        fh = [l for l in range(nfh) if 32 * l < tw]
        sw = [nfh + g for g in range(ns) if g < ngrp]
        v2 = [nfh + ns + l for l in range(12) if sum(32 * l + 384 * j < wv for j in range(cols)) == 2]
        v1 = [nfh + ns + l for l in range(12) if sum(32 * l + 384 * j < wv for j in range(cols)) == 1]
        classes = [fh, sw, v2, v1]
        work = set(fh + sw + v2 + v1)
        idle = [l for l in range(24) if l not in work]
        counts = [len(x) for x in classes]
        cands = list(layouts(counts))
        print(f"# {cfg}: tile {c['tile']} cols {cols} working FH/S/V2/V1 {counts}, {len(cands)} layouts, default map "
              f"{c['warp_map']}", flush=True)
        if len(cands) > maxc:
            cands = random.sample(cands, maxc)
        x = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        y = torch.empty((H, W), dtype=torch.float32, device="cuda")
        a = b.make_args(repair_threshold=-1.0)
        fl = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        def time_map(m, n):
            if m is None:
                os.environ.pop("BF_WMAP_OVERRIDE", None)
            else:
                os.environ["BF_WMAP_OVERRIDE"] = ",".join(map(str, m))
            ts = []
            for i in range(n + 1):
                fl.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                b.apply_ex(plan, x.data_ptr(), y.data_ptr(), 1, H, W, s, a)
                e1.record()
                e1.synchronize()
                if i >= 1:
                    ts.append(e0.elapsed_time(e1))
            return statistics.median(ts)

        n1 = 2 if cfg == "cfg4" else 5
        time_map(None, 3)
        ref = y.clone()
        t_def = time_map(None, 3 * n1)
        t_id = time_map(list(range(24)), 3 * n1)
        print(f"{cfg} default {t_def:.4f} ms identity {t_id:.4f} ms", flush=True)
        res = []
        for sub in cands:
            m = build_map(sub, classes, idle, (0, 1, 2, 3))
            res.append((time_map(m, n1), sub))
        res.sort()
        print(f"{cfg} best 12 of {len(res)} (first pass):")
        for t, sub in res[:12]:
            print(f"  {t:.4f} {sub}")
        print("ALL " + json.dumps({"cfg": cfg, "counts": counts, "results": [[round(t, 5), sub] for t, sub in res]}))
        print(f"{cfg} worst 3:")
        for t, sub in res[-3:]:
            print(f"  {t:.4f} {sub}")
        # second pass: the best layouts, more runs, several role orders inside a sub-partition
        best = []
        for t, sub in res[:6]:
            for order in ((0, 1, 2, 3), (1, 0, 2, 3), (2, 3, 1, 0), (2, 3, 0, 1), (1, 2, 3, 0)):
                for idle_at in (None, 0, 2):
                    m = build_map(sub, classes, idle, order, idle_at)
                    t2 = time_map(m, 4 * n1)
                    assert torch.equal(y, ref), "a warp map changed the output"
                    best.append((t2, sub, (order, idle_at), m))
        best.sort(key=lambda r: r[0])
        print(f"{cfg} second pass:")
        for t2, sub, order, m in best[:10]:
            print(f"  {t2:.4f} {sub} order {order} map {m}")
        print(json.dumps({"cfg": cfg, "default_ms": t_def, "identity_ms": t_id, "best_ms": best[0][0],
                          "best_layout": best[0][1], "best_order": best[0][2], "best_map": best[0][3]}), flush=True)


if __name__ == "__main__":
    main()
