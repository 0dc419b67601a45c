"""Design tool (not a test, not the oracle): error budget of the GPU number format at single,
ill-conditioned pixels of a full-size config (cfg4's den / sum K~_s ~ 4e-4 pixels).

Emulates kernel 2b's arithmetic for one output pixel bit-faithfully (fp32 polynomial base angle,
fp32 rotation recurrence, per-tap rint quantisation with the box weight folded into the scale,
exact int vertical sums, U' = (U + urnd) >> ush, exact int horizontal box sums, F = sum_b
mulhi(H_b, ax_b), fp64 combine weights rounded to int, exact int64 num / den) and switches the
error sources off one at a time, against the oracle's value of the same pixel.

    python tools/numerics_pixel.py cfg4 8191,4624 8191,2997 1,5654
"""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import bf, fit  # noqa: E402
from synth import CONFIGS, config_input, config_params  # noqa: E402
from tools.numerics_v6 import axis_boxes, poly_base  # noqa: E402

f32 = np.float32


def fma32(a, b, c):
    return (np.asarray(a, np.float64) * np.asarray(b, np.float64) + np.asarray(c, np.float64)).astype(f32)


def emulate(I, plan, y0, x0, mode):
    """out(y0, x0) in the kernel's number format (mode switches error sources off)."""
    H, W = I.shape
    D = plan.D
    r = plan.radius
    boxes = axis_boxes(plan)                     # [(lo, hi, w)] nested, symmetric (same on both axes)
    rows = np.arange(max(0, y0 - r), min(H, y0 + r + 1))
    cols = np.arange(max(0, x0 - r), min(W, x0 + r + 1))
    win = I[np.ix_(rows, cols)].astype(np.float64)
    v = rows - y0
    u = cols - x0
    wmax = max(abs(w) for _, _, w in boxes)
    # vertical quantisation: scale per box, q bits as large as int32 allows (host quantise())
    wsum = sum(abs(w) / wmax * (hi - lo + 1) for lo, hi, w in boxes)
    qb = 22
    while qb > 8 and math.ldexp(wsum, qb) + 4.0 * (boxes[0][1] - boxes[0][0] + 8) >= 2147483647.0 - 65536.0:
        qb -= 1
    qs = [f32(math.ldexp(w / wmax, qb)) for _, _, w in boxes]
    qsD = [f32(float(q) / D) for q in qs]
    ubound = sum((abs(float(q)) + 0.5) * (hi - lo + 1) for q, (lo, hi, _) in zip(qs, boxes))
    nxmax = max(hi - lo + 1 for lo, hi, _ in boxes)
    ush = 0
    while (ubound / 2.0 ** ush + 1.0) * nxmax >= 2147483000.0:
        ush += 1
    urnd = (1 << (ush - 1)) if ush else 0
    uprime = ubound / 2.0 ** ush + 1.0
    rw = sum(abs(w) / wmax * (hi - lo + 1) for lo, hi, w in boxes)
    abits = 30
    while abits > 16 and uprime * rw * 2.0 ** (abits - 32) + 8.0 >= 2147483000.0:
        abits -= 1
    ax = [int(round(math.ldexp(w / wmax, abits))) for _, _, w in boxes]
    asum = sum(abs(a) for a in plan.rng.a)
    amax = max(abs(a) for a in plan.rng.a)
    wbits = 29
    while wbits > 8 and (math.ldexp(asum, wbits) * 2.0 * 2147483648.0 >= 4.0e18 or math.ldexp(amax, wbits) >= 2.0e9):
        wbits -= 1
    # channels of the taps
    I32 = win.astype(f32)
    if mode.get("exact_channels"):
        th = math.pi * win / D
    else:
        c1, s1 = poly_base(I32, D)
    inbox = [((v >= lo) & (v <= hi))[:, None] for lo, hi, _ in boxes]
    ck, sk = np.ones_like(I32), np.zeros_like(I32)
    kcur = 0
    # pixel's fp64 weights (Cheb recurrence ~ exact cos / sin)
    thx = math.pi * float(I[y0, x0]) / D
    num = 0.0 if mode.get("float_combine") else 0
    den = 0.0 if mode.get("float_combine") else 0
    for k, a in zip(plan.rng.k, plan.rng.a):
        if mode.get("exact_channels"):
            gc, gs = np.cos(k * th), np.sin(k * th)
        else:
            while kcur < k:
                ck, sk = fma32(sk, -s1, (ck * c1).astype(f32)), fma32(ck, s1, (sk * c1).astype(f32))
                kcur += 1
            gc, gs = ck.astype(np.float64), sk.astype(np.float64)
        F = []
        for X, useI in ((gc, False), (gs, False), (gc, True), (gs, True)):
            Ucol = np.zeros(len(cols), dtype=np.float64 if (mode.get("exact_quant") or mode.get("exact_quant_kernel_channels")) else np.int64)
            for bi, (q, qd) in enumerate(zip(qs, qsD)):
                mult = (qd * I32).astype(f32).astype(np.float64) if useI else float(q)
                if mode.get("exact_quant"):
                    t = X * (win / D * float(q) if useI else float(q))
                elif mode.get("exact_quant_kernel_channels"):
                    t = X * mult
                else:
                    t = np.rint(X * mult).astype(np.int64)
                Ucol = Ucol + np.sum(np.where(inbox[bi], t, 0), axis=0)
            if mode.get("exact_quant") or mode.get("no_ush_round") or mode.get("exact_quant_kernel_channels"):
                Up = (Ucol + 0.0) / 2.0 ** ush
            else:
                Up = (Ucol + urnd) >> ush
            Fv = 0.0 if mode.get("exact_F") else 0
            for (lo, hi, _), a_ in zip(boxes, ax):
                Hb = Up[(u >= lo) & (u <= hi)].sum()
                if mode.get("exact_F"):
                    Fv += float(Hb) * a_ / 2.0 ** 32
                elif mode.get("round_F"):
                    Fv += (int(Hb) * a_ + (1 << 31)) >> 32
                else:
                    Fv += (int(Hb) * a_) >> 32
            F.append(Fv)
        wc_f = a * math.cos(k * thx) * 2.0 ** wbits
        ws_f = a * math.sin(k * thx) * 2.0 ** wbits
        if mode.get("exact_w"):
            wc, wsn = wc_f, ws_f
        else:
            wc, wsn = int(round(wc_f)), int(round(ws_f))
        if mode.get("float_combine") or mode.get("exact_w") or mode.get("exact_F"):
            den = den + float(wc) * F[0] + float(wsn) * F[1]
            num = num + float(wc) * F[2] + float(wsn) * F[3]
        else:
            den += wc * F[0] + wsn * F[1]
            num += wc * F[2] + wsn * F[3]
    return D * float(num) / float(den) if den > 0 else float(I[y0, x0])


MODES = {
    "kernel (round 1)": {},
    "F exact (no mulhi truncation)": {"exact_F": True},
    "F rounded (mad.wide + 2^31)": {"round_F": True},
    "U' unrounded": {"no_ush_round": True},
    "weights unrounded": {"exact_w": True},
    "F exact + U' unrounded": {"exact_F": True, "no_ush_round": True},
    "F exact + U' unrounded + w exact": {"exact_F": True, "no_ush_round": True, "exact_w": True},
    "exact channels (fp64 cos)": {"exact_channels": True},
    "exact channels + exact quant": {"exact_channels": True, "exact_quant": True, "exact_F": True, "exact_w": True},
    "only tap quantisation": {"exact_channels": True, "exact_F": True, "no_ush_round": True, "exact_w": True},
    "only fp32 channels": {"exact_quant_kernel_channels": True, "exact_F": True, "no_ush_round": True,
                           "exact_w": True},
}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    pts = [tuple(int(t) for t in s.split(",")) for s in sys.argv[2:]] or [(8191, 4624)]
    spec = CONFIGS[cfg]
    p = config_params(spec)
    plan = fit.make_plan(**p)
    r = spec.radius
    full = None
    for (y, x) in pts:
        if full is None:
            full = config_input(spec)
        ya, yb = max(0, y - 2 * r), min(spec.H, y + 2 * r + 1)
        xa, xb = max(0, x - 2 * r), min(spec.W, x + 2 * r + 1)
        crop = full[ya:yb, xa:xb]
        yc, xc = y - ya, x - xa
        ref, num, den = bf.bf_direct(crop, plan, pixels=[(yc, xc)])
        mass = fit.spatial_kernel_values(plan.sp)
        print(f"{cfg} pixel ({y},{x}): oracle {ref[0]:.6f}  den {den[0]:.3e}", flush=True)
        for name, m in MODES.items():
            o = emulate(crop, plan, yc, xc, m)
            print(f"   {name:40s} out {o:.6f}  err {abs(o - ref[0]) * 255 / plan.D:.2e}", flush=True)


if __name__ == "__main__":
    main()
