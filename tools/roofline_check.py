"""Cross-check of bench.py's algorithmic roofline against the hardware: from an ncu
--set full report, the FADD + FMUL + FFMA thread-instructions each kernel executed per
cycle per SMSP as a fraction of the FMA pipe's 32 lanes (what `peak` counts).  The
algorithmic fraction (bench.py roofline.frac, counted from the method's required work)
must not exceed it.

  python tools/roofline_check.py gpurun_out/prof.ncu-rep [profiles/<tag>_bench_cfg5.json]
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep = sys.argv[1]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        tot = 0.0
        for op in ("fadd", "ffma", "fmul"):
            tot += float(d[f"smsp__sass_thread_inst_executed_op_{op}_pred_on.avg.per_cycle_elapsed"])
        q = "ffc" if "(int)1" in d["Kernel Name"] or "<1," in d["Kernel Name"] else "motval"
        out[q] = {"kernel": d["Kernel Name"], "fp32_thread_ops_per_cycle_per_smsp": tot,
                  "fma_pipe_fp32_utilisation": tot / 32.0}
    if len(sys.argv) > 2:
        b = json.load(open(sys.argv[2]))
        k = b["roofline"]["kernel"].split("<")[1].rstrip(">")
        out["bench_algorithmic_frac"] = {"kernel": k, "frac": b["roofline"]["frac"],
                                         "executed_fma_pipe_frac": out.get(k, {}).get("fma_pipe_fp32_utilisation")}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
