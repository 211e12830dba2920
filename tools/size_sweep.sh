#!/bin/bash
# Throughput vs batch size on one GPU (cfg5 motion prefixes): where does a shard saturate?
# (the driver's strong-scaling run gives each of 8 GPUs 131,072 motions)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for M in 16384 32768 65536 131072 262144 524288 1048576 2097152 4194304; do
  timeout 600 python bench.py --motions $M --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$M.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep_$M.json')); b=d['breakdown']; print($M, d['value'], d['ms_per_step'], b['motval_ms'], b['ffc_ms'])"
done
