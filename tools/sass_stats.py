"""Per-kernel SASS statistics of a built library (instruction count, load/store mix):
  python tools/sass_stats.py [lib.so] [name-substring ...]"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_23960_b200/libmrv.so"
want = sys.argv[2:]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)[1:]
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if want and not any(w in name for w in want):
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(?:\.[A-Z0-9_.]+)?", f)
    c = Counter(ins)
    mem = {k: c[k] for k in ("LDS", "LD", "LDG", "STS", "ST", "STG", "LDL", "STL") if c[k]}
    print(f"{name}: {len(ins)} instr, {mem}")
