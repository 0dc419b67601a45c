"""Print the SASS of the kernels whose mangled name contains every given substring, with an
opcode histogram.  Usage: python tools/sass_of.py LIB SUBSTR... [--hist]"""
import collections
import re
import subprocess
import sys

lib, subs = sys.argv[1], [a for a in sys.argv[2:] if not a.startswith("--")]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if all(s in name for s in subs):
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", b)
        print(name, len(ops), "instructions")
        if "--hist" in sys.argv:
            for op, n in collections.Counter(o.split(".")[0] for o in ops).most_common(25):
                print(f"  {op:10s} {n}")
        else:
            print(b)
