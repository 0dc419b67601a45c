"""Summarise an ncu --set full report at the SASS level: executed instructions per opcode,
warp-stall samples per reason, and the hottest instructions.  Usage:
    python tools/ncu_sass_summary.py report.ncu-rep [top_n]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    idx = {n: i for i, n in enumerate(h)}
    stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    by_op = collections.Counter()
    samp_op = collections.Counter()
    stalls = collections.Counter()
    tot = 0
    recs = []
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        src = r[idx["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        opb = op.split(".")[0]
        n = int(r[idx["Instructions Executed"]] or 0)
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        by_op[opb] += n
        samp_op[opb] += s
        tot += n
        for c in stall_cols:
            stalls[c] += int(r[idx[c]] or 0)
        recs.append((s, n, r[idx["Address"]], src))
    print(f"total warp-instructions executed: {tot:,}")
    print("\nopcode          executed   share   stall-samples")
    ts = sum(samp_op.values()) or 1
    for op, n in by_op.most_common(30):
        print(f"{op:12s} {n:14,d} {100*n/tot:6.1f}% {100*samp_op[op]/ts:6.1f}%")
    print("\nstall reason samples")
    tt = sum(stalls.values()) or 1
    for c, n in stalls.most_common(12):
        print(f"{c:28s} {100*n/tt:6.1f}%")
    print(f"\ntop {top} instructions by samples")
    for s, n, a, src in sorted(recs, reverse=True)[:top]:
        print(f"{s:7d} {n:12,d} {a[-5:]} {src[:90]}")


if __name__ == "__main__":
    main()


def buckets(rep):
    """executed warp-instructions grouped by per-instruction execution count (one group ~ one loop)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
    h = rows[0]
    idx = {n: i for i, n in enumerate(h)}
    g = collections.defaultdict(lambda: [0, 0, 0, collections.Counter(), collections.Counter()])
    stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        n = int(r[idx["Instructions Executed"]] or 0)
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        src = r[idx["Source"]].strip().split()
        op = (src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "?")).split(".")[0]
        e = g[n]
        e[0] += 1
        e[1] += n
        e[2] += s
        e[3][op] += 1
        for c in stall_cols:
            e[4][c[6:]] += int(r[idx[c]] or 0)
    tot = sum(v[1] for v in g.values())
    print("\nexec-count  #instr  total-executed  share  samples  top opcodes")
    for n, (ni, te, ss, ops, st) in sorted(g.items(), key=lambda kv: -kv[1][2])[:12]:
        print(f"{n:>11,d} {ni:6d} {te:15,d} {100*te/tot:5.1f}% {ss:8d}  {dict(ops.most_common(6))}")
        sst = sum(st.values()) or 1
        print("              stalls: " + ", ".join(f"{k} {100*v/sst:.0f}%" for k, v in st.most_common(5)))


if __name__ == "__main__" and len(sys.argv) > 1:
    buckets(sys.argv[1])
