#!/bin/bash
# ncu --set full capture (with source) of the MotVal + FFC kernels on a cfg5 slice.
# Usage via gpurun: bash tools/ncu_full.sh <tag> [motions] [config]
tag=${1:-prof}; M=${2:-262144}; CFG=${3:-cfg5}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
timeout 300 python bench.py --config $CFG --motions $M --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_plain.json 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:mrv_query_kernel -c 2 \
  -o gpurun_out/${tag} python bench.py --config $CFG --motions $M --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/${tag}_ncu.log
tail -2 gpurun_out/${tag}_ncu.log
