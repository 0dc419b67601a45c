"""Runs one config through a given build of libbf.so a few times (for ncu captures of diagnostic
builds): python tools/run_lib.py LIB cfg [reps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1803_00004_b200._bf as b  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402

b.LIB_PATH = os.path.abspath(sys.argv[1])
spec = CONFIGS[sys.argv[2]]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = config_params(spec)
img = config_input(spec)
if img.ndim == 3:
    img = img[0]
u8 = img.dtype.name == "uint8"
plan = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
              radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
              input_dtype="u8" if u8 else "f32")
H, W = img.shape
x = torch.from_numpy(np.ascontiguousarray(img)).cuda()
y = torch.empty((H, W), dtype=torch.float32, device="cuda")
ws = b.workspace_size(plan, H, W)
wsb = torch.empty(max(ws, 1), dtype=torch.uint8, device="cuda")
a = b.make_args(workspace=(wsb.data_ptr(), ws) if ws else (0, 0), repair_threshold=-1.0)
for _ in range(reps):
    b.apply_ex(plan, x.data_ptr(), y.data_ptr(), 1, H, W, torch.cuda.current_stream().cuda_stream, a)
torch.cuda.synchronize()
print("ok", sys.argv[1], sys.argv[2])
