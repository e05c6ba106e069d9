#!/bin/bash
# Round-2 evidence set for the current C3 bench step (one GPU; run under gpurun):
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
  --csv --log-file gpurun_out/r2_launches_c3.csv python bench.py $ARGS > gpurun_out/r2_launches_c3.log 2>&1
tail -2 gpurun_out/r2_launches_c3.log
full r2_prof_gemm_layer "gemm2_kernelILi256ELb0" 4 4      # qkv, o, up, down of primary layer 1 (bf16 CTA-pair kernel)
full r2_prof_fa "fa_sparse_row" 3 1
full r2_prof_tf32_layer "gemm2_kernelILi128ELb1" 4 4       # scoring-model layer 1 (3xTF32 CTA-pair kernel)
full r2_prof_banked_tc "banked_tc" 3 1
full r2_prof_norm "embed_rmsnorm|rmsnorm" 60 1
full r2_prof_asm "assemble_kernel" 0 1
ls -la gpurun_out
