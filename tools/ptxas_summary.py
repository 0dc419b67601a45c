"""Compile csrc/bf_kernels.cu with -Xptxas -v and print registers / spills per instantiation."""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "paper_1803_00004_b200/csrc/bf_kernels.cu"
r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
                    "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", "-o", "/tmp/_k.o", src],
                   capture_output=True, text=True)
name = None
for line in (r.stdout + r.stderr).splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"(bf_\w+?_kernel)I(.*)EEEv", name)
        name = (k.group(1) + "<" + re.sub(r"L[ib](\d+)E", r"\1,", k.group(2) + "E").rstrip(",") + ">") if k else name
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = f"spill st {m.group(1)} ld {m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{name:48s} regs {m.group(1):>4s}  {spill}")
    if "error" in line:
        print(line)
