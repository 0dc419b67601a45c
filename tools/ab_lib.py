"""A/B device timing of two builds of libbf.so on one config (CUDA events, L2 flushed):
    python tools/ab_lib.py LIB_A LIB_B [cfg] [env=value ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import CONFIGS, config_input, config_params  # noqa: E402


import ctypes  # noqa: E402

_CDLL = ctypes.CDLL


class _Tolerant:
    """CDLL proxy: symbols an older build lacks resolve to a stub (the A/B calls only bf_apply)."""

    def __init__(self, path):
        self._L = _CDLL(path)
        self._stubs = {}

    def __getattr__(self, name):
        try:
            return getattr(self._L, name)
        except AttributeError:
            return self._stubs.setdefault(name, type("Stub", (), {})())


def run(lib_path, cfg):
    import paper_1803_00004_b200._bf as b
    b._lib = None
    b.C.CDLL = _Tolerant
    b.LIB_PATH = lib_path
    spec = CONFIGS[cfg]
    p = config_params(spec)
    img = config_input(spec)
    u8 = img.dtype.name == "uint8"
    plan = b.Plan(spatial=p["spatial"], range_kind=p["range_kind"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                  radius=p["radius"], n_terms=p["n_terms"], intensity_max=p["intensity_max"],
                  input_dtype="u8" if u8 else "f32")
    x = torch.from_numpy(img).cuda()
    y = torch.empty(img.shape, dtype=torch.float32, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for i in range(8):
        flush.zero_()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        b.apply(plan, x.data_ptr(), y.data_ptr(), img.shape[0], img.shape[1], s)
        e.record()
        e.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(e))
    return statistics.median(ts), y.cpu()


if __name__ == "__main__":
    cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg4"
    for kv in sys.argv[4:]:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    ta, ya = run(sys.argv[1], cfg)
    tb, yb = run(sys.argv[2], cfg)
    print(f"{cfg}: A {ta:.3f} ms  B {tb:.3f} ms  max|A-B| {float((ya - yb).abs().max()):.3e}")
