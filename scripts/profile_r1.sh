#!/bin/bash
# ncu evidence for the timed region of bench.py (one GPU). Run under gpurun.
set -x
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu"
# every launch of one timed step with its device time
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
  --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/launches_bench.log 2>&1
# full sets: the bf16 tcgen05 GEMM (MLP-size) and the sparse-row attention
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  -k regex:"gemm_kernelILi256ELb0" -s 4 -c 2 -o gpurun_out/prof_gemm python bench.py $ARGS > gpurun_out/prof_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  -k regex:"sparse_row_attention" -c 1 -o gpurun_out/prof_attn python bench.py $ARGS > gpurun_out/prof_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  -k regex:"assemble_kernel" -c 1 -o gpurun_out/prof_asm python bench.py $ARGS > gpurun_out/prof_asm.log 2>&1
ls -la gpurun_out
