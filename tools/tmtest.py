import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1803_00004_b200 as b
from synth import CONFIGS, config_input, config_params
which = sys.argv[1]
spec = CONFIGS[which.split('_')[0]]; p = config_params(spec); img = config_input(spec)
if img.ndim == 3: img = img[0]
dt = "u8" if img.dtype == np.uint8 else "f32"
if which.endswith('_f32'): img = img.astype(np.float32); dt = "f32"
n = int(sys.argv[2]) if len(sys.argv) > 2 else p["n_terms"]
pl = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], radius=p["radius"], n_terms=n, intensity_max=p["intensity_max"], input_dtype=dt)
print(which, n, b.config(pl, *img.shape), flush=True)
t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
o = b.bilateral_filter(pl, t, repair_threshold=-1.0); torch.cuda.synchronize(); print("ok", float(o.double().mean()), flush=True)
