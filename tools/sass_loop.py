"""Static SASS summary of the hot loop of a kernel in libtpgpu.so.

usage: python tools/sass_loop.py REGEX   -- prints instruction count per
function and the opcode mix of the largest backward-branch loop."""
import re
import subprocess
import sys
from collections import Counter

so = "paper_2502_21013_b200/libtpgpu.so"
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
pat = re.compile(sys.argv[1])
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if not pat.search(name):
        continue
    ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", f)
    addr = [(int(a, 16), t.strip()) for a, t in ins]
    # loops: backward BRA
    best = None
    for a, t in addr:
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        mm = re.search(r"BRA .*?(0x[0-9a-f]+)", t)
        if mm:
            tgt = int(mm.group(1), 16)
            if tgt < a and (best is None or a - tgt > best[1] - best[0]):
                best = (tgt, a)
    print(name[:140], "total", len(addr))
    if best:
        body = [t for a, t in addr if best[0] <= a <= best[1]]
        c = Counter()
        for t in body:
            op = t.split()[0]
            if op.startswith("@"):
                op = t.split()[1]
            c[op.split(".")[0]] += 1
        print("  loop", len(body), dict(c.most_common(16)))
