#!/bin/bash
# One GPU session: build, GPU tests, smoke, default bench, ncu launch list of the same
# command.  Usage (from the repo root, via gpurun): bash tools/gpu_check.sh [tag]
tag=${1:-chk}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench exit $?" >> gpurun_out/${tag}_bench.err
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/${tag}_ncu.log 2>&1
  echo "ncu exit $?" >> gpurun_out/${tag}_ncu.log
fi
tail -3 gpurun_out/${tag}_pytest.log gpurun_out/${tag}_smoke.log
cat gpurun_out/${tag}_bench.json
