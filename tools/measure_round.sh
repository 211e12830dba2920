#!/bin/bash
# One GPU session of round measurements (via gpurun): bash tools/measure_round.sh <tag>
#   <tag>_bench_<cfg>.json   default bench line per config (cfg5 = the driver's default) + pp5
#   <tag>_launches.csv       ncu launch list (gpu__time_duration.sum) of the default bench command
#   <tag>_traffic.csv        ncu DRAM bytes per launch of the production kernels at FULL size
#                            (cfg5, 2^20 motions: no scaling) -> profiles/ncu_traffic.json
tag=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/${tag}_bench_cfg5.json 2> gpurun_out/${tag}_bench_cfg5.err
echo "cfg5 exit $?"
for c in cfg1 cfg2 cfg3 cfg4 pp5; do
  timeout 600 python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  echo "$c exit $?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py > gpurun_out/${tag}_launches.log 2>&1
echo "launch list exit $?"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:mrv_query_kernel -c 6 --csv --log-file gpurun_out/${tag}_traffic.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-roofline-nee > gpurun_out/${tag}_traffic.log 2>&1
echo "traffic exit $?"
