"""Per-source-line / per-stage attribution of an ncu --set full report (pc sampling +
executed instructions), by joining ncu's SASS source page with nvdisasm line info.

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep [--lib paper_2604_23960_b200/libmrv.so] [--top 40]

The library must be the exact build that was profiled (same source, same flags).
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# kernels.cu line ranges -> stage names (first line of each region; regions end at the next)
STAGES = [
    (1, "misc"), (122, "predicates"), (166, "interp"), (195, "sincos"), (207, "se3_pose"), (241, "robot_fk"),
    (316, "warp_state"), (353, "frame_sink"), (403, "load_frame"), (414, "robot_fk_dh"), (449, "fk_stage"),
    (481, "pack_round"), (507, "seg_helpers"), (550, "flush_env"), (594, "env_pass"), (643, "flush_narrow"),
    (705, "self"), (780, "env_stage"), (802, "flush_l1"), (908, "rr_stage"), (979, "process_item"),
    (1096, "stage_scene"), (1130, "kernel_main"), (1175, "fk_export"),
]


def stage_of(line):
    name = "?"
    for l0, n in STAGES:
        if line >= l0:
            name = n
    return name


def sass_lines(lib, mangled):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.startswith("kernels") and "scene" not in f][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    out, cur, line, infile = {}, None, 0, False
    for l in txt.splitlines():
        m = re.match(r"\.text\.(\S+):", l)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            infile = m.group(1).endswith("kernels.cu")
            line = int(m.group(2)) if infile else -int(m.group(2))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m and cur == mangled:
            out[int(m.group(1), 16)] = (line, m.group(2).strip())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2604_23960_b200", "libmrv.so"))
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'^"Kernel Name",', txt, flags=re.M)[1:]
    src = open(os.path.join(ROOT, "paper_2604_23960_b200", "csrc", "kernels.cu")).read().splitlines()
    for b in blocks:
        name = b.splitlines()[0].strip().strip(",").strip('"')
        q = 1 if "(int)1" in name else 0
        cnt = 1 if "(bool)1" in name else 0
        mangled = f"_ZN3mrv16mrv_query_kernelILi{q}ELb{cnt}EEEvNS_7KParamsE"
        rows = list(csv.reader(io.StringIO("\n".join(b.splitlines()[1:]))))
        hdr = rows[0]
        ia, isamp, iexec = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
            "Instructions Executed")
        recs = [r for r in rows[1:] if len(r) == len(hdr)]
        base = int(recs[0][ia], 16)
        lines = sass_lines(a.lib, mangled)
        by_line = collections.Counter()
        by_line_i = collections.Counter()
        by_stage = collections.Counter()
        by_stage_i = collections.Counter()
        tot_s = tot_i = 0
        for r in recs:
            off = int(r[ia], 16) - base
            s, i = float(r[isamp] or 0), float(r[iexec] or 0)
            ln = lines.get(off, (0, ""))[0]
            by_line[ln] += s
            by_line_i[ln] += i
            st = stage_of(ln) if ln > 0 else "header"
            by_stage[st] += s
            by_stage_i[st] += i
            tot_s += s
            tot_i += i
        print(f"== {name}: {tot_s:.0f} samples, {tot_i:.3e} warp instructions")
        print("stage               samples%   instr%")
        for st, s in by_stage.most_common():
            print(f"  {st:18s} {100 * s / tot_s:6.1f}   {100 * by_stage_i[st] / tot_i:6.1f}")
        print("top lines (samples%, instr%, line, source)")
        for ln, s in by_line.most_common(a.top):
            code = src[ln - 1].strip()[:90] if 0 < ln <= len(src) else f"(header line {-ln})"
            print(f"  {100 * s / tot_s:5.1f} {100 * by_line_i[ln] / tot_i:5.1f}  {ln:5d}  {code}")


if __name__ == "__main__":
    main()
