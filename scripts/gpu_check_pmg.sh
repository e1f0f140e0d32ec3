#!/bin/bash
# ncu evidence for the SURVEY.md §8f kernels (p-multigrid, Schwarz/FDM,
# projection): one full capture per kernel family from a V-cycle at E=20^3,
# N=7 (RAS, FP64 and FP32 local solves) and the launch list of one pMG solve.
# usage: bash scripts/gpu_check_pmg.sh <tag>
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"fdm_kernel|schwarz_post|interp3|cheb_step|dense_matvec|gs_classes" -c 14 \
  -o gpurun_out/pmg_full_$TAG python scripts/prof_vcycle.py --counts 20 20 20 --smoother ras --precision 64 \
  > gpurun_out/ncu_pmg_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"fdm_kernel" -c 1 \
  -o gpurun_out/fdm32_full_$TAG python scripts/prof_fdm.py --precision 32 --reps 2 \
  > gpurun_out/ncu_fdm32_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"multi_wdot|multi_axpy" -c 4 \
  -o gpurun_out/proj_full_$TAG python scripts/projection_bench.py --steps 3 \
  > gpurun_out/ncu_proj_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/pmg_launches_$TAG.csv python scripts/pmg_bench.py --counts 20 20 20 \
  --smoothers ras > /dev/null 2>&1
tail -1 gpurun_out/ncu_pmg_$TAG.log gpurun_out/ncu_fdm32_$TAG.log gpurun_out/ncu_proj_$TAG.log
ls gpurun_out
