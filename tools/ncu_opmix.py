"""Executed-instruction mix by SASS opcode of each kernel in an ncu --set full report.

  python tools/ncu_opmix.py gpurun_out/prof.ncu-rep [--top 30]
"""
import argparse
import collections
import csv
import io
import re
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    seen = set()
    for b in re.split(r'^"Kernel Name",', txt, flags=re.M)[1:]:
        name = b.splitlines()[0].strip().strip(",").strip('"')
        if name in seen:
            continue
        seen.add(name)
        rows = list(csv.reader(io.StringIO("\n".join(b.splitlines()[1:]))))
        hdr = rows[0]
        isrc, iexec = hdr.index("Source"), hdr.index("Instructions Executed")
        mix = collections.Counter()
        tot = 0.0
        for r in rows[1:]:
            if len(r) != len(hdr):
                continue
            ins = r[isrc].strip()
            if ins.startswith("@"):
                ins = ins.split(None, 1)[1] if " " in ins else ins
            op = ins.split()[0].split(".")[0] if ins else "?"
            n = float(r[iexec] or 0)
            mix[op] += n
            tot += n
        print(f"== {name}: {tot:.3e} warp instructions")
        for op, n in mix.most_common(a.top):
            print(f"  {op:10s} {100 * n / tot:5.1f} %")


if __name__ == "__main__":
    main()
