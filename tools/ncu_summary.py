"""Summarise an ncu report (``--set full``) and/or a launch list into profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep --name r1 [--launches gpurun_out/launches.csv]
      [--config cfg5] [--motions 262144]

Writes profiles/<name>_ncu_summary.md (per-kernel duration, occupancy, issue,
pipe utilisation, stall mix, DRAM bytes); with --traffic it also merges the per-launch
DRAM traffic, scaled from the profiled motion count to the config's full size, into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic -- normally written from
a full-size launch list by tools/traffic_json.py instead).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__occupancy_limit_shared_mem", "block limit (smem)"),
    ("launch__occupancy_limit_registers", "block limit (regs)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.avg.per_cycle_elapsed", "FFMA thread-ops / cycle / SMSP"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.avg.per_cycle_elapsed", "FADD thread-ops / cycle / SMSP"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.avg.per_cycle_elapsed", "FMUL thread-ops / cycle / SMSP"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst executed %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe inst executed %"),
    ("dram__bytes_read.sum.per_second", "DRAM read throughput"),
    ("sm__cycles_elapsed.avg", "elapsed cycles (per SM)"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0}


def val_si(k, key):
    v = num(k.get(key))
    u = k["_units"].get(key, "")
    return None if v is None else v * SCALE.get(u, 1.0)


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--name", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--motions", type=int, default=262144)
    ap.add_argument("--full-motions", type=int, default=1 << 20)
    ap.add_argument("--traffic", action="store_true", help="merge scaled DRAM bytes into profiles/ncu_traffic.json")
    a = ap.parse_args()
    kernels = raw(a.rep)
    lines = [f"# ncu summary `{a.name}` ({os.path.basename(a.rep)})", "",
             f"Profiled command: bench.py on {a.config} with {a.motions} motions; ncu --set full --clock-control none.", ""]
    traffic = {}
    for k in kernels:
        name = k.get("Kernel Name", "?")
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in KEYS:
            if key in k:
                lines.append(f"| {label} (`{key}`) | {k[key]} {k['_units'].get(key, '')} |")
        stalls = sorted(((num(v) or 0.0, kk) for kk, v in k.items()
                         if kk.startswith("smsp__pcsamp_warps_issue_stalled") and not kk.endswith("not_issued")),
                        reverse=True)
        tot = sum(s for s, _ in stalls) or 1.0
        lines.append("")
        lines.append("Stall mix (pc sampling): " + ", ".join(
            f"{kk.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * s / tot:.0f}%" for s, kk in stalls[:7]))
        lines.append("")
        rd, wr = val_si(k, "dram__bytes_read.sum"), val_si(k, "dram__bytes_write.sum")
        if rd is not None and wr is not None:
            q = "motval" if "<0," in name or "(int)0" in name else "ffc"
            traffic[q] = (rd + wr) * a.full_motions / a.motions
    if a.launches:
        lines += ["## Launch list (gpu__time_duration.sum, cold-cache, serialised)", "", "| id | kernel | ns |", "|---|---|---|"]
        with open(a.launches) as f:
            txt = "".join(l for l in f if not l.startswith("=="))
        for r in csv.DictReader(io.StringIO(txt)):
            lines.append(f"| {r.get('ID')} | {r.get('Kernel Name', '')[:70]} | {r.get('Metric Value')} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    out = os.path.join(ROOT, "profiles", f"{a.name}_ncu_summary.md")
    open(out, "w").write("\n".join(lines) + "\n")
    if not a.traffic:
        print(out, traffic)
        return 0
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj.setdefault(a.config, {}).update(traffic)
    tj["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from an ncu --set full capture, scaled "
                   "linearly from the profiled motion count to the config's full size")
    json.dump(tj, open(tp, "w"), indent=1)
    print(out, traffic)


if __name__ == "__main__":
    sys.exit(main())
