#!/bin/bash
# Round-2 profiling recipe (one GPU): the launch list of the bench command's
# timed region, then `ncu --set full` captures of the quantizer (sta_q shape:
# K=1152, LN + 3 outputs, 16384 rows) and the u8 GEMM (16384 x 1152 x 1152)
# at the north_star target's per-video size.  Each command first runs plain.
set -x
OUT=gpurun_out
python bench.py --no-extra --no-cpu-baseline --steps 1 --warmup 1 > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
QC_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/launches_r02.csv python bench.py --no-extra --no-cpu-baseline --steps 1 --warmup 1 \
    > $OUT/ncu_launches.log 2>&1
python tools/quant_bench.py --cases qkv_ln --iters 2 > $OUT/qb_plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on \
    -k regex:"aq4_pass1|aq2_pass2_hot|init_keys" -s 3 -c 3 -o $OUT/r02_quant \
    python tools/quant_bench.py --cases qkv_ln --iters 2 > $OUT/ncu_quant.log 2>&1
python tools/gemm_bench.py --shapes 1152x1152 --iters 2 > $OUT/gb_plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on \
    -k regex:"gemm_u8" -s 3 -c 1 -o $OUT/r02_gemm \
    python tools/gemm_bench.py --shapes 1152x1152 --iters 2 > $OUT/ncu_gemm.log 2>&1
exit 0
