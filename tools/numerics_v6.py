"""Design tool (not a test, not the oracle): bit-faithful numpy emulation of candidate kernel
number formats, scored against the fp64 oracle on crops of the BASELINE configs.

V   vertical box sums: 'sep' = exact int sums per box, U' = (sum_b ay_b S_b) >> sh (kernel v5);
    'fold' = the box weight folded into the per-tap quantisation scale, one exact int state
    U = sum_b sum_v rint(w_b X), U' = round(U / 2^sh).
gen channel generation from an fp32 base angle: 'exact' (correctly rounded fp32 cos(k th)),
    'rot' (rotation recurrence), 'cheb' (Chebyshev three-term recurrence, fp32 FMA).
H   exact int box sums of U', F = round((sum_b ax_b H_b) / 2^fs)  (27-bit ax).
C   W = rint(fp32(a_k 2^wbits) * c) (F2I) or the 22-bit FFMA magic; exact int64 num/den.
"""
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import bf, fit  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402

f32 = np.float32


def fma32(a, b, c):
    return (np.asarray(a, np.float64) * np.asarray(b, np.float64) + np.asarray(c, np.float64)).astype(f32)


def box1d(q, lo, hi, axis):
    """exact sum of q over offsets lo..hi along axis (zero outside)."""
    q = np.asarray(q, dtype=np.int64)
    n = q.shape[axis]
    c = np.cumsum(q, axis=axis)
    c = np.concatenate([np.zeros_like(np.take(c, [0], axis=axis)), c], axis=axis)
    idx = np.arange(n)
    a = np.clip(idx + hi + 1, 0, n)
    b = np.clip(idx + lo, 0, n)
    return np.take(c, a, axis=axis) - np.take(c, b, axis=axis)


def rshift_round(x, sh):
    if sh <= 0:
        return x
    return (x + (1 << (sh - 1))) >> sh


def axis_boxes(plan):
    """separable factor f(u) = sum_b w_b [lo_b <= u <= hi_b] from the lowered kernel."""
    K = fit.spatial_kernel_values(plan.sp)
    r = plan.radius
    f = K[r] / math.sqrt(K[r, r])
    boxes = []
    # peel nested symmetric boxes from the outside in
    lev = 0.0
    for u in range(-r, 1):
        if abs(f[u + r] - lev) > 1e-15 * abs(f[r]):
            boxes.append((u, -u, f[u + r] - lev))
            lev = f[u + r]
    fk = np.zeros(2 * r + 1)
    for lo, hi, w in boxes:
        fk[lo + r:hi + r + 1] += w
    assert np.allclose(np.outer(fk, fk), K, atol=1e-14), "not separable"
    return boxes


PS = [3.141592741e+00, -5.167712688e+00, 2.550163269e+00, -5.992513299e-01, 8.204647899e-02, -7.022163365e-03]
PQ = [1.000000000e+00, -4.934802055e+00, 4.058712006e+00, -1.335262775e+00, 2.353305817e-01, -2.580653690e-02,
      1.927883714e-03, -1.004332444e-04]


def poly_base(I32, D):
    """fp32 emulation of the kernel's base angle: t' = I/D - 1/2 as fma(I, invD_hi, -0.5) + I*invD_lo,
    sin(pi t') = t' P(t'^2), cos(pi t') = Q(t'^2) (Horner, FMA), then cos(pi t) = -sin(pi t'),
    sin(pi t) = cos(pi t')."""
    invD = 1.0 / D
    hi = f32(invD)
    lo = f32(invD - float(hi))
    t = fma32(I32, hi, f32(-0.5))
    t = (t + (I32 * lo).astype(f32)).astype(f32)
    z = (t * t).astype(f32)
    p = np.full_like(z, f32(PS[-1]))
    for c in PS[-2::-1]:
        p = fma32(p, z, f32(c))
    q = np.full_like(z, f32(PQ[-1]))
    for c in PQ[-2::-1]:
        q = fma32(q, z, f32(c))
    return (-(p * t)).astype(f32), q


def sim(I, plan, mode):
    D = plan.D
    I64 = np.asarray(I, np.float64)
    I32 = I64.astype(f32)
    H, W = I.shape
    boxes = axis_boxes(plan)
    wmax = max(abs(w) for _, _, w in boxes)
    QB = mode.get("qbits", 22)
    # vertical quantisation scales / integer weights
    if mode["V"] == "fold":
        sc = [f32(w / wmax * 2.0 ** QB) for _, _, w in boxes]
        ubound = sum(abs(w) / wmax * 2.0 ** QB * (hi - lo + 1) for lo, hi, w in boxes)
    else:
        ay = [int(round(w / wmax * 2 ** 27)) for _, _, w in boxes]
        sbound = sum(abs(a) * (2.0 ** QB) * (hi - lo + 1) for a, (lo, hi, _) in zip(ay, boxes))
        ubound = sbound
    nxmax = max(hi - lo + 1 for lo, hi, _ in boxes)
    ush = 0
    while (ubound / 2.0 ** ush + 1) * nxmax >= 2 ** 31 - 1:
        ush += 1
    ax = [int(round(w / wmax * 2 ** 27)) for _, _, w in boxes]
    fb = sum(abs(a) * (ubound / 2.0 ** ush + 1) * (hi - lo + 1) for a, (lo, hi, _) in zip(ax, boxes))
    fsh = 0
    while fb / 2.0 ** fsh >= 2 ** 31 - 1:
        fsh += 1
    # base angle fp32 (correctly rounded)
    th = math.pi * I64 / D
    c1, s1 = np.cos(th).astype(f32), np.sin(th).astype(f32)
    if mode.get("poly"):
        c1, s1 = poly_base(I32, D)
    num = np.zeros((H, W), dtype=object) if mode.get("bigint") else np.zeros((H, W), np.int64)
    den = np.zeros_like(num)
    wbits = mode.get("wbits", 29)
    gen = mode.get("gen", "rot")
    ck, sk = np.ones_like(c1), np.zeros_like(s1)
    cprev, sprev = None, None
    kcur = 0
    for k, a in zip(plan.rng.k, plan.rng.a):
        while kcur < k:
            if gen == "rot":
                ck, sk = fma32(ck, c1, -(sk * s1)), fma32(sk, c1, ck * s1)
            elif gen == "cheb":
                if kcur == 0:
                    cn, sn = c1.copy(), s1.copy()
                else:
                    cn, sn = fma32(f32(2) * c1, ck, -cprev), fma32(f32(2) * c1, sk, -sprev)
                cprev, sprev = ck, sk
                ck, sk = cn, sn
            kcur += 1
        if gen == "exact":
            gc, gs = np.cos(math.pi * k * I64 / D).astype(f32), np.sin(math.pi * k * I64 / D).astype(f32)
        else:
            gc, gs = ck, sk
        Fs = []
        for X, useI in ((gc, False), (gs, False), (gc, True), (gs, True)):
            if mode["V"] == "fold":
                U = np.zeros((H, W), np.int64)
                for (lo, hi, w), s in zip(boxes, sc):
                    mult = (f32(s / f32(D)) * I32).astype(f32) if useI else s
                    q = np.rint(X.astype(np.float64) * np.asarray(mult, np.float64)).astype(np.int64)
                    U += box1d(q, lo, hi, 0)
                Up = rshift_round(U + 0, ush)
            else:
                s = f32(2.0 ** QB)
                mult = (f32(s / f32(D)) * I32).astype(f32) if useI else s
                q = np.rint(X.astype(np.float64) * np.asarray(mult, np.float64)).astype(np.int64)
                acc = np.zeros((H, W), np.int64)
                for a_, (lo, hi, _) in zip(ay, boxes):
                    acc += a_ * box1d(q, lo, hi, 0)
                Up = rshift_round(acc, ush)
            Fv = np.zeros((H, W), np.int64)
            for a_, (lo, hi, _) in zip(ax, boxes):
                Fv += a_ * box1d(Up, lo, hi, 1)
            Fs.append(rshift_round(Fv, fsh))
        if mode.get("w64"):
            wc = np.rint(a * 2.0 ** wbits * np.cos(math.pi * k * I64 / D)).astype(np.int64)
            ws = np.rint(a * 2.0 ** wbits * np.sin(math.pi * k * I64 / D)).astype(np.int64)
        elif mode.get("w22"):
            aw = f32(a * 2.0 ** 22 / max(abs(x) for x in plan.rng.a))
            wc = np.rint(gc.astype(np.float64) * float(aw)).astype(np.int64)
            ws = np.rint(gs.astype(np.float64) * float(aw)).astype(np.int64)
        else:
            aw = f32(a * 2.0 ** wbits)
            wc = np.rint((gc * aw).astype(f32)).astype(np.int64)
            ws = np.rint((gs * aw).astype(f32)).astype(np.int64)
        den = den + wc * Fs[0] + ws * Fs[1]
        num = num + wc * Fs[2] + ws * Fs[3]
    numf = np.asarray(num, np.float64)
    denf = np.asarray(den, np.float64)
    out = np.where(denf > 0, (D * numf / np.where(denf > 0, denf, 1)).astype(f32), I32).astype(np.float64)
    return out, dict(ush=ush, fsh=fsh)


def main():
    cfgs = sys.argv[1:] or ["cfg0", "cfg2", "cfg3", "cfg4"]
    for cfg in cfgs:
        spec = CONFIGS[cfg]
        p = config_params(spec)
        plan = fit.make_plan(**p)
        if cfg in ("cfg2", "cfg4"):
            side = 1024 if cfg == "cfg2" else 2048
            full = config_input(spec, H=side, W=side)
            n = 333 if cfg == "cfg2" else 420
            I = full[100:100 + n, 200:200 + n]
        else:
            I = config_input(spec, H=256, W=256)
        t = time.time()
        ref, num, den, _ = bf.bf_box(I, plan, return_parts=True)
        Ksum = fit.spatial_kernel_values(plan.sp).sum()
        scale = 255.0 / plan.D
        print(f"{cfg}: {I.shape} oracle {time.time()-t:.1f}s  min den/sumK = {np.min(den)/Ksum:.2e}", flush=True)
        modes = {
            "sep  rot  w29 (v5)": dict(V="sep", gen="rot"),
            "fold rot  w29": dict(V="fold", gen="rot"),
            "fold cheb w29": dict(V="fold", gen="cheb"),
            "fold exact w29": dict(V="fold", gen="exact"),
            "fold cheb w22": dict(V="fold", gen="cheb", w22=True),
            "fold rot  w22": dict(V="fold", gen="rot", w22=True),
        }
        for name, m in modes.items():
            try:
                out, info = sim(I, plan, m)
            except AssertionError as e:
                print("   ", name, "skipped:", e)
                continue
            e = np.abs(out - ref) * scale
            print(f"   {name:22s} max {e.max():.2e}  rmse {np.sqrt(np.mean(e*e)):.2e}  {info}", flush=True)


if __name__ == "__main__":
    main()
