"""Diagnostic / A-B builds of libbf.so: recompiles the given translation units with extra nvcc
flags into _obj_var/NAME and links them with the product objects into tools/var/libbf_NAME.so.

    python tools/build_variant.py NAME "-DBF_X_NOFH=1" [bf_k_ws2.cu ...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_00004_b200 import build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2].split()
    tus = sys.argv[3:] or ["bf_k_ws2.cu"]
    B.build()
    od = os.path.join(ROOT, "_obj_var", name)
    os.makedirs(od, exist_ok=True)
    os.makedirs(os.path.join(ROOT, "tools", "var"), exist_ok=True)

    def comp(src):
        obj = os.path.join(od, os.path.splitext(src)[0] + ".o")
        cmd = [B.nvcc(), *B.NVCC_FLAGS, *flags, "-c", "-o", obj, os.path.join(B.CSRC, src)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return src, obj

    with ThreadPoolExecutor(max_workers=len(tus)) as ex:
        done = dict(ex.map(comp, tus))
    objs = [done.get(s, os.path.join(B.OBJ, os.path.splitext(s)[0] + ".o")) for s in B.SOURCES]
    out = os.path.join(ROOT, "tools", "var", f"libbf_{name}.so")
    subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-lcudart"],
                   check=True)
    print(out)


if __name__ == "__main__":
    main()
