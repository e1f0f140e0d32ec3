#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list, ncu full captures.
# usage: bash scripts/gpu_check.sh <tag> [skip-tests]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu_$TAG.log
  tail -3 gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-ceiling > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bk5_ -s 3 -c 1 \
  -o gpurun_out/bk5_full_$TAG python bench.py --steps 2 --warmup 3 --no-bp5 --no-cpu --no-ceiling > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pcg|gs_classes|cg_update" -s 30 -c 3 \
  -o gpurun_out/cg_full_$TAG python bench.py --steps 2 --warmup 3 --no-cpu --no-ceiling > gpurun_out/ncu_cg_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log gpurun_out/ncu_cg_$TAG.log
ls gpurun_out
