import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1803_00004_b200._bf as b
b.LIB_PATH = sys.argv[1]
from synth import CONFIGS, config_input, config_params
spec = CONFIGS["cfg0"]; p = config_params(spec); img = config_input(spec)
pl = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], radius=p["radius"], n_terms=8, intensity_max=p["intensity_max"], input_dtype="u8")
t = torch.from_numpy(np.ascontiguousarray(img)).cuda(); y = torch.empty(img.shape, dtype=torch.float32, device="cuda")
a = b.make_args(repair_threshold=-1.0)
b.apply_ex(pl, t.data_ptr(), y.data_ptr(), 1, 256, 256, 0, a)
torch.cuda.synchronize(); print("ok")
