#!/bin/bash
# ncu full captures of the kernels below the roofline (one GPU; run under gpurun)
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu"
N="--kernel-name-base mangled"
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" $N \
  -k regex:"banked_f32_kernel" -s 3 -c 1 -o gpurun_out/prof_banked python bench.py $ARGS > gpurun_out/prof_banked.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" $N \
  -k regex:"gemm_kernelILi256ELb1" -s 2 -c 1 -o gpurun_out/prof_tf32 python bench.py $ARGS > gpurun_out/prof_tf32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" $N \
  -k regex:"embed_rmsnorm" -s 60 -c 2 -o gpurun_out/prof_norm python bench.py $ARGS > gpurun_out/prof_norm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" $N \
  -k regex:"fa_sparse_row" -s 3 -c 1 -o gpurun_out/prof_fa2 python bench.py $ARGS > gpurun_out/prof_fa2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" $N \
  -k regex:"gemm_kernelILi256ELb0" -s 4 -c 1 -o gpurun_out/prof_gemm python bench.py $ARGS > gpurun_out/prof_gemm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
  --csv --log-file gpurun_out/launches_v2.csv python bench.py $ARGS > gpurun_out/launches_v2.log 2>&1
ls -la gpurun_out
