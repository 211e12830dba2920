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

# stage = the kernels.cu function a source line falls in (located by its definition line)
MARKERS = [
    ("misc", None), ("predicates", "bool sph_sph("), ("interp", "struct Interp"), ("sincos", "void fast_sincos("),
    ("se3_pose", "void se3_pose("), ("robot_fk", "void robot_fk(const SV"), ("warp_state", "struct Counters"),
    ("frame_sink", "struct FrameSink"), ("load_frame", "void load_frame("), ("robot_fk_dh", "void robot_fk_dh("),
    ("fk_stage", "void fk_stage("), ("pack_round", "struct Pack"), ("seg_helpers", "uint32_t seg_idx("),
    ("flush_env", "uint32_t flush_env("), ("env_grid", "bool env_grid_pass("), ("pp_access", "const float4* pp_row("), ("capsule", "void frame_pt("), ("flush_narrow", "uint32_t flush_narrow("),
    ("self", "bool flush_self("), ("env_stage", "bool env_stage("), ("flush_l1", "bool flush_l1("),
    ("rr_swept", "uint32_t rr_stage_swept("), ("rr_tile", "uint32_t rr_stage_tile("), ("rr_stage", "uint32_t rr_stage("), ("fk_env_fused", "uint32_t fk_env_fused("), ("process_item", "void set_batch("), ("run_spread", "void run_spread("), ("stage_scene", "uint32_t smem_u32("),
    ("kernel_main", "void __launch_bounds__"), ("fk_export", "struct OutSink"),
]


def stage_table(src):
    out = [(1, "misc")]
    for name, pat in MARKERS[1:]:
        for i, l in enumerate(src):
            if pat in l:
                # include the template line / comment block directly above
                j = i
                while j > 0 and (src[j - 1].startswith("template") or src[j - 1].startswith("//")):
                    j -= 1
                out.append((j + 1, name))
                break
    return sorted(out)


STAGES = []


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
    STAGES[:] = stage_table(src)
    seen = set()
    for b in blocks:
        name = b.splitlines()[0].strip().strip(",").strip('"')
        tm = re.search(r"\(int\)(\d+), \(bool\)(\d+)", name)
        q, cnt = int(tm.group(1)), int(tm.group(2))
        if name in seen:
            continue
        seen.add(name)
        targs = re.findall(r"\((int|bool)\)(\d+)", name.split("(mrv::KParams)")[0])
        mangled = "_ZN3mrv16mrv_query_kernelI" + "".join(("Li" if t == "int" else "Lb") + v + "E" for t, v in targs) + \
            "EEvNS_7KParamsE"
        rows = list(csv.reader(io.StringIO("\n".join(b.splitlines()[1:]))))
        hdr = rows[0]
        ia, isamp, iexec = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
            "Instructions Executed")
        recs = [r for r in rows[1:] if len(r) == len(hdr)]
        reasons = ["stall_selected", "stall_wait", "stall_short_sb", "stall_long_sb", "stall_not_selected",
                   "stall_branch_resolving", "stall_no_inst", "stall_math", "stall_mio", "stall_dispatch"]
        ri = {k: hdr.index(k) for k in reasons if k in hdr}
        by_stage_r = collections.defaultdict(collections.Counter)
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
            for k, ix in ri.items():
                by_stage_r[st][k] += float(r[ix] or 0)
            tot_s += s
            tot_i += i
        print(f"== {name}: {tot_s:.0f} samples, {tot_i:.3e} warp instructions")
        short = {"stall_selected": "sel", "stall_wait": "wait", "stall_short_sb": "shsb", "stall_long_sb": "lgsb",
                 "stall_not_selected": "nsel", "stall_branch_resolving": "br", "stall_no_inst": "noi",
                 "stall_math": "math", "stall_mio": "mio", "stall_dispatch": "disp"}
        print("stage               samples%   instr%   " + " ".join(f"{short[k]:>5s}" for k in ri))
        for st, s in by_stage.most_common():
            print(f"  {st:18s} {100 * s / tot_s:6.1f}   {100 * by_stage_i[st] / tot_i:6.1f}   " +
                  " ".join(f"{100 * by_stage_r[st][k] / tot_s:5.1f}" for k in ri))
        print("top lines (samples%, instr%, line, source)")
        for ln, s in by_line.most_common(a.top):
            code = src[ln - 1].strip()[:90] if 0 < ln <= len(src) else f"(header line {-ln})"
            print(f"  {100 * s / tot_s:5.1f} {100 * by_line_i[ln] / tot_i:5.1f}  {ln:5d}  {code}")


if __name__ == "__main__":
    main()
