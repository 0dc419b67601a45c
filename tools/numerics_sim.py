"""Design tool (not a test, not the oracle): simulate candidate GPU arithmetic in numpy and
report the error against the fp64 oracle, to choose the kernel's number formats.

Pipeline simulated (the design in DESIGN.md):
  channels X in fp32 (rotation recurrence or correctly rounded), quantised to int fixed point
  with 22 bits of full scale; vertical 2-box sums exact in integers; U = V_r + g V_rin in fp32;
  U quantised to int (22 bits of its bound); horizontal 2-box sums exact; F = H_r + g H_rin;
  combine with weights in fp64 (or fp32), divide.
"""
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import bf, fit  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402


def box1d(q, e, axis):
    """exact integer box sum of half-width e along axis (zero outside)."""
    q = np.asarray(q, dtype=np.int64)
    n = q.shape[axis]
    c = np.cumsum(q, axis=axis)
    c = np.concatenate([np.zeros_like(np.take(c, [0], axis=axis)), c], axis=axis)
    idx = np.arange(n)
    hi = np.clip(idx + e + 1, 0, n)
    lo = np.clip(idx - e, 0, n)
    return np.take(c, hi, axis=axis) - np.take(c, lo, axis=axis)


def sim(I, plan, cfg_r, mode):
    D = plan.D
    r = plan.radius
    rin = (2 * r + 1) // 4
    # 1-D factor f = alpha on |u|<=r, alpha+beta on |u|<=rin -> scale so f = 1 + gamma*[|u|<=rin]
    Ks = fit.spatial_kernel_values(plan.sp)
    f = Ks[r] / math.sqrt(Ks[r, r])
    single = np.ptp(f) < 1e-12
    alpha = f[0]
    gamma = 0.0 if single else (f[r] - f[0]) / f[0]
    I64 = np.asarray(I, dtype=np.float64)
    I32 = I64.astype(np.float32)
    H, W = I.shape
    num = np.zeros((H, W))
    den = np.zeros((H, W))
    qbits = mode.get("qbits", 22)
    # base angle for the rotation recurrence (fp32, correctly rounded from exact)
    th1 = np.pi * I64 / D
    c1 = np.cos(th1).astype(np.float32)
    s1 = np.sin(th1).astype(np.float32)
    ck = np.ones_like(c1)
    sk = np.zeros_like(s1)
    kprev = 0
    ks = list(plan.rng.k)
    for k, a in zip(ks, plan.rng.a):
        if mode.get("rotation"):
            while kprev < k:
                ck, sk = (ck * c1 - sk * s1).astype(np.float32), (sk * c1 + ck * s1).astype(np.float32)
                kprev += 1
            gc32, gs32 = ck, sk
        else:
            gc32 = np.cos(np.pi * k * I64 / D).astype(np.float32)
            gs32 = np.sin(np.pi * k * I64 / D).astype(np.float32)
        chans = [(gc32 * I32).astype(np.float32), (gs32 * I32).astype(np.float32), gc32, gs32]
        bounds = [D, D, 1.0, 1.0]
        F = []
        for X, bnd in zip(chans, bounds):
            if k == 0 and X is gs32 or (k == 0 and bnd == D and X is chans[1]):
                F.append(np.zeros((H, W)))
                continue
            sc = (2.0 ** qbits - 1) / bnd
            q = np.rint(X.astype(np.float64) * sc).astype(np.int64)
            if mode.get("fp32_channels_no_quant"):
                q = X.astype(np.float64)
                Vr = bf.box_sum(bf.sat2d(q), 0, 0, -r, r)
                Vi = bf.box_sum(bf.sat2d(q), 0, 0, -rin, rin)
                U = (Vr + gamma * Vi)
                Hr = bf.box_sum(bf.sat2d(U), -r, r, 0, 0)
                Hi = bf.box_sum(bf.sat2d(U), -rin, rin, 0, 0)
                F.append(alpha * alpha * (Hr + gamma * Hi))
                continue
            Vr = box1d(q, r, 0)
            Vi = box1d(q, rin, 0) if not single else 0
            U = (Vr.astype(np.float32) + np.float32(gamma) * np.asarray(Vi, dtype=np.float32)).astype(np.float32)
            Ubound = (2 * r + 1 + gamma * (2 * rin + 1)) * (2.0 ** qbits)
            su = (2.0 ** mode.get("ubits", 22) - 1) / Ubound
            uq = np.rint(U.astype(np.float64) * su).astype(np.int64)
            Hr = box1d(uq, r, 1)
            Hi = box1d(uq, rin, 1) if not single else 0
            if mode.get("F32"):
                Fv = (Hr.astype(np.float32) + np.float32(gamma) * np.asarray(Hi, dtype=np.float32)).astype(np.float64)
            else:
                Fv = Hr.astype(np.float64) + gamma * np.asarray(Hi, dtype=np.float64)
            F.append(Fv * (alpha * alpha / (sc * su)))
        if mode.get("w64"):
            wc, ws = np.cos(np.pi * k * I64 / D), np.sin(np.pi * k * I64 / D)
        else:
            wc, ws = gc32.astype(np.float64), gs32.astype(np.float64)
        if mode.get("combine32"):
            num = (num + np.float32(a) * (wc.astype(np.float32) * F[0].astype(np.float32) + ws.astype(np.float32) * F[1].astype(np.float32))).astype(np.float32)
            den = (den + np.float32(a) * (wc.astype(np.float32) * F[2].astype(np.float32) + ws.astype(np.float32) * F[3].astype(np.float32))).astype(np.float32)
        else:
            num += a * (wc * F[0] + ws * F[1])
            den += a * (wc * F[2] + ws * F[3])
    out, fb = bf.normalise(I64, np.asarray(num, np.float64), np.asarray(den, np.float64))
    return out


def main():
    cfgs = sys.argv[1:] or ["cfg0", "cfg2", "cfg4"]
    for cfg in cfgs:
        spec = CONFIGS[cfg]
        p = config_params(spec)
        plan = fit.make_plan(**p)
        if cfg in ("cfg2", "cfg4"):
            full = config_input(spec, H=1024 if cfg == "cfg2" else 2048, W=1024 if cfg == "cfg2" else 2048)
            n = 256 if cfg == "cfg2" else 420
            I = full[100:100 + n, 200:200 + n]
        else:
            I = config_input(spec, H=256, W=256)
        t = time.time()
        ref, num, den, _ = bf.bf_box(I, plan, return_parts=True)
        Ksum = fit.spatial_kernel_values(plan.sp).sum()
        scale = 255.0 / plan.D
        print(f"{cfg}: {I.shape} oracle {time.time()-t:.1f}s  min den/sumK = {np.min(den)/Ksum:.2e}")
        modes = {
            "fp32 ch (no quant), fp64 sums, w32": {"fp32_channels_no_quant": True},
            "int22 exact, F64, w32": {},
            "int22 exact, F64, w64": {"w64": True},
            "int22 exact, F32, w64": {"F32": True, "w64": True},
            "int22 rot32, F64, w64": {"rotation": True, "w64": True},
            "int22 rot32, F64, w32": {"rotation": True},
            "int22 rot32, F32, w32": {"rotation": True, "F32": True},
            "int22, combine32": {"combine32": True},
        }
        for name, m in modes.items():
            out = sim(I, plan, spec.radius, m)
            e = np.abs(out - ref) * scale
            print(f"   {name:36s} max {e.max():.2e}  rmse {np.sqrt(np.mean(e*e)):.2e}")


if __name__ == "__main__":
    main()
