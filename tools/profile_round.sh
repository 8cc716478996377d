#!/bin/bash
# Profiling evidence for profiles/ (run on the GPU box from the repo root, after
# the same commands have exited 0 without ncu):
#   1. launch list of the bench command's timed region (cold-cache, serialised)
#   2. ncu --set full of one quantizer call (ln1 site shape) and one u8 GEMM
set -u
mkdir -p gpurun_out
QC_PROFILE_RANGE=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum \
  --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"aq4_pass1|aq2_pass2|init_keys" -f -o gpurun_out/quant \
  python tools/quant_bench.py --cases ln1 --iters 1 > gpurun_out/ncu_quant.log 2>&1
echo "quant capture rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:gemm_u8_tcgen05 -c 1 -f -o gpurun_out/gemm \
  python tools/gemm_bench.py --M 8192 --shapes 1152x1152 --iters 1 > gpurun_out/ncu_gemm.log 2>&1
echo "gemm capture rc=$?"
