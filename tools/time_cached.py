"""Device time of bf_apply_cached (cfg2, Case 1 cache of k < 17, repair off) for several builds
of libbf.so, one process per build: python tools/time_cached.py LIB [LIB ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, statistics, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1803_00004_b200._bf as b
b.LIB_PATH = LIB
from synth import CONFIGS, config_input, config_params
spec = CONFIGS["cfg2"]; p = config_params(spec); img = config_input(spec)
plan = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
              radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"], input_dtype="f32")
H, W = img.shape
x = torch.from_numpy(img).cuda(); y = torch.empty((H, W), dtype=torch.float32, device="cuda")
n = b.cache_size(plan, 17, H, W); buf = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
d = b.precompute(plan, 17, x.data_ptr(), H, W, buf.data_ptr(), n, s)
a = b.make_args(repair_threshold=-1.0)
fl = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ts = []
for i in range(15):
    fl.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.apply_cached(plan, d, buf.data_ptr(), x.data_ptr(), y.data_ptr(), s, a); e1.record(); e1.synchronize()
    if i >= 3: ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
gb = (16 * 16 + 8) * H * W / 1e9
print(f"{os.path.basename(LIB)} apply_cached {ms:.4f} ms  {gb / ms:.0f} GB/s  sum(out)={float(y.double().sum()):.6f}", flush=True)
'''
for lib in sys.argv[1:]:
    code = f"ROOT={ROOT!r}\nLIB={os.path.abspath(lib)!r}\n" + CHILD
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
    sys.stdout.write(r.stdout or r.stderr[-1500:])
