"""Repaired / fallback pixel counts and the repair pass's share of the step per config (GPU)."""
import statistics
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_00004_b200 as b  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402

for cfg in sys.argv[1].split(","):
    spec = CONFIGS[cfg]
    p = config_params(spec)
    img = config_input(spec)
    if img.ndim == 3:
        img = img[int(sys.argv[2]) if len(sys.argv) > 2 else 0]
    u8 = img.dtype.name == "uint8"
    plan = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                  radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                  input_dtype="u8" if u8 else "f32")
    H, W = img.shape
    x = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    y = torch.empty((H, W), dtype=torch.float32, device="cuda")
    ws = b.workspace_size(plan, H, W)
    wsb = torch.empty(max(ws, 1), dtype=torch.uint8, device="cuda")
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    rep = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for thr in (0.0, -1.0):
        a = b.make_args(workspace=(wsb.data_ptr(), ws) if ws else (0, 0), repair_threshold=thr,
                        fallback_count=fb.data_ptr(), repaired_count=rep.data_ptr())
        ts = []
        for i in range(5):
            fb.zero_()
            rep.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.apply_ex(plan, x.data_ptr(), y.data_ptr(), 1, H, W, s, a)
            e1.record()
            e1.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        print(f"{cfg} threshold {thr}: {statistics.median(ts):.3f} ms repaired {int(rep.item())} fallback {int(fb.item())}",
              flush=True)
