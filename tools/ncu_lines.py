"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo):
    python tools/ncu_lines.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, out = None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            out.append((int(r[4] or 0), int(r[7] or 0), cur, r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
out.sort(reverse=True)
print(f"{'stall%':>6} {'warp-inst':>14}  line")
for s, e, f, ln, src in out[:n]:
    print(f"{s * 100 / tot:6.1f} {e:>14}  {f}:{ln}  {src.strip()}")
