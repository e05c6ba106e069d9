#!/bin/bash
# Round-1 evidence set for the current C3 bench step (one GPU; run under gpurun):
# launch list of one timed step + ncu --set full of the top kernels.
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu"
N="--kernel-name-base mangled"
full() {  # $1 = out name, $2 = kernel regex, $3 = skip, $4 = count
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" $N \
    -k regex:"$2" -s $3 -c $4 -o gpurun_out/$1 python bench.py $ARGS > gpurun_out/$1.log 2>&1
  tail -2 gpurun_out/$1.log
}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
  --csv --log-file gpurun_out/launches_c3.csv python bench.py $ARGS > gpurun_out/launches_c3.log 2>&1
tail -2 gpurun_out/launches_c3.log
full prof_gemm_layer "gemm2_kernel" 4 4      # qkv, o, up, down of primary layer 1 (CTA-pair kernel)
full prof_fa "fa_sparse_row" 3 1
full prof_tf32_layer "gemm_kernelILi.*ELb1" 4 4       # scoring-model layer 1
full prof_banked_tc "banked_tc" 3 1
full prof_norm "embed_rmsnorm|rmsnorm" 60 1
full prof_asm "assemble_kernel" 0 1
ls -la gpurun_out
# our CTA-pair GEMM vs cuBLAS on one 8192^3 bf16 GEMM (side by side)
timeout 600 ncu --set full --clock-control none --kernel-name-base mangled -c 2 -o gpurun_out/prof_gemm_vs_cublas \
  python scripts/gemm_pair_ncu.py > gpurun_out/prof_gemm_vs_cublas.log 2>&1
tail -2 gpurun_out/prof_gemm_vs_cublas.log
