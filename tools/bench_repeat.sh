#!/bin/bash
# Run-to-run spread of the default bench line (N = 1): 5 fresh processes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/rep_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rep_$i.json')); print($i, d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
