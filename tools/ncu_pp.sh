#!/bin/bash
# ncu --set full capture of the PP-ST-RRT kernel (pp5 slice).  Usage via gpurun: bash tools/ncu_pp.sh <tag> [motions]
tag=${1:-pp}; M=${2:-262144}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mrv_query_kernel -c 1 \
  -o gpurun_out/${tag} python bench.py --config pp5 --motions $M --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu exit $?"
