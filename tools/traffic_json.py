"""profiles/ncu_traffic.json from an ncu DRAM-bytes launch list of the production kernels at
full size (tools/measure_round.sh <tag>_traffic.csv): bytes read + written per launch, the
median over the captured launches of each query's lean instance.

  python tools/traffic_json.py gpurun_out/<tag>_traffic.csv [config]"""
import csv
import io
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg5"
txt = "".join(l for l in open(path) if not l.startswith("=="))
rows = list(csv.DictReader(io.StringIO(txt)))
per = {}
for r in rows:
    name = r.get("Kernel Name", "")
    q = "motval" if "<(int)0" in name or "<0," in name else "ffc"
    key = (r.get("ID"), q)
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
    if r["Metric Name"].startswith("dram__bytes") and scale:
        per.setdefault(key, 0.0)
        per[key] += v * scale
out = {}
for q in ("motval", "ffc"):
    vals = [v for (i, qq), v in per.items() if qq == q]
    if vals:
        out[q] = statistics.median(vals)
p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
d = json.load(open(p)) if os.path.exists(p) else {}
d[cfg] = out
d["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the production (lean) kernels, measured by "
              "ncu on the full-size launch (tools/measure_round.sh), median over the captured launches")
json.dump(d, open(p, "w"), indent=1)
print(json.dumps(d, indent=1))
