# round-2 GPU call 8: where the scoring pass and the low-ratio (default 8/5
# rule) path spend their time: ncu --set full of the four 3xTF32 GEMM shapes,
# GEMM microbench, launch lists of the default-rule step at 5% and 20%
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/bench_gemm.py > gpurun_out/r8_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 4 \
  -o gpurun_out/r8_tf32 python scripts/bench_gemm.py --only tf32 --reps 1 --trials 1 > gpurun_out/r8_tf32_ncu.log 2>&1
OUT=r8_launches_dr05 BENCHARGS="--ratio 0.05 --window-threshold 5 --no-sweep" sh scripts/launch_list.sh
OUT=r8_launches_dr20 BENCHARGS="--ratio 0.2 --window-threshold 5 --no-sweep" sh scripts/launch_list.sh
echo done
