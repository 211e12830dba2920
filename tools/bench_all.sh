#!/bin/bash
# Default bench line for every config (N = 1) -> gpurun_out/<tag>_bench_<cfg>.json
tag=${1:-all}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  echo "$c exit $?"
done
