#!/bin/bash
# ncu --set full of one primary attention launch at recompute ratios 5 % and
# 40 % (C3 step): low ratios move toward the HBM-bound regime (few query rows
# per key tile), high ratios stay tensor-bound. One GPU, under gpurun.
mkdir -p gpurun_out
for r in 0.05 0.4; do
  timeout 900 ncu --set full --clock-control none --kernel-name-base mangled --nvtx --nvtx-include "timed/" \
    -k regex:fa_sparse_row -s 3 -c 1 -o gpurun_out/prof_fa_r$r \
    python bench.py --steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu --ratio $r > gpurun_out/prof_fa_r$r.log 2>&1
  tail -1 gpurun_out/prof_fa_r$r.log
done
