"""Device time of the fused kernel (no repair pass) for several builds of libbf.so, one process
per build (CUDA events, L2 flushed, median of 12):
    python tools/time_libs.py cfg2,cfg4 LIB [LIB ...]
Prints one line per (config, lib) and max|out - out(first lib)|."""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, statistics, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1803_00004_b200._bf as b
b.LIB_PATH = LIB
from synth import CONFIGS, config_input, config_params
for cfg in CFGS:
    spec = CONFIGS[cfg]; p = config_params(spec); img = config_input(spec)
    if img.ndim == 3: img = img[0]
    u8 = img.dtype.name == "uint8"
    plan = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                  radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"], input_dtype="u8" if u8 else "f32")
    H, W = img.shape
    x = torch.from_numpy(np.ascontiguousarray(img)).cuda(); y = torch.empty((H, W), dtype=torch.float32, device="cuda")
    ws = b.workspace_size(plan, H, W); wsb = torch.empty(max(ws, 1), dtype=torch.uint8, device="cuda")
    a = b.make_args(workspace=(wsb.data_ptr(), ws) if ws else (0, 0), repair_threshold=-1.0)
    fl = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    n = 6 if cfg == "cfg4" else 15
    for i in range(n):
        fl.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.apply_ex(plan, x.data_ptr(), y.data_ptr(), 1, H, W, s, a); e1.record(); e1.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    np.save(OUT + "_" + cfg + ".npy", y.cpu().numpy())
    print(f"{cfg} {os.path.basename(LIB)} {statistics.median(ts):.4f} ms", flush=True)
'''


def main():
    cfgs = sys.argv[1].split(",")
    libs = sys.argv[2:]
    import numpy as np
    outs = []
    for i, lib in enumerate(libs):
        out = f"/tmp/tl_{i}"
        code = f"ROOT={ROOT!r}\nLIB={os.path.abspath(lib)!r}\nCFGS={cfgs!r}\nOUT={out!r}\n" + CHILD
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
        sys.stdout.write(r.stdout)
        if r.returncode:
            sys.stdout.write(r.stderr[-2000:])
        outs.append(out)
    for cfg in cfgs:
        try:
            ref = np.load(outs[0] + "_" + cfg + ".npy")
        except OSError:
            continue
        for lib, o in zip(libs[1:], outs[1:]):
            try:
                d = float(np.abs(np.load(o + "_" + cfg + ".npy") - ref).max())
                print(f"{cfg} {os.path.basename(lib)} max|diff| vs {os.path.basename(libs[0])}: {d:.3e}")
            except OSError:
                pass


if __name__ == "__main__":
    main()
