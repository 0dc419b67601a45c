"""End-to-end time of bf_apply_host (pinned host buffers, copies inside) for several builds of
libbf.so, one process per build:  python tools/time_host.py cfg2 LIB [LIB ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time, statistics, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1803_00004_b200._bf as b
b.LIB_PATH = LIB
from synth import CONFIGS, config_input, config_params
spec = CONFIGS[CFG]; p = config_params(spec); img = config_input(spec)
if img.ndim == 3: img = img[0]
u8 = img.dtype.name == "uint8"
plan = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
              radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"], input_dtype="u8" if u8 else "f32")
H, W = img.shape
torch.cuda.init()
h_in = torch.from_numpy(np.ascontiguousarray(img)).pin_memory()
h_out = torch.empty((H, W), dtype=torch.float32).pin_memory()
s = torch.cuda.current_stream().cuda_stream
ts = []
for i in range(25):
    t0 = time.perf_counter(); b.apply_host(plan, h_in.data_ptr(), h_out.data_ptr(), H, W, s); t = time.perf_counter() - t0
    if i >= 5: ts.append(t)
print(f"{CFG} {os.path.basename(LIB)} e2e median {statistics.median(ts)*1e3:.4f} ms min {min(ts)*1e3:.4f} ms  {H*W/1e6/statistics.median(ts):.0f} MP/s", flush=True)
'''
cfg = sys.argv[1]
for lib in sys.argv[2:]:
    code = f"ROOT={ROOT!r}\nLIB={os.path.abspath(lib)!r}\nCFG={cfg!r}\n" + CHILD
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    sys.stdout.write(r.stdout)
    if r.returncode:
        sys.stdout.write(r.stderr[-1500:])
