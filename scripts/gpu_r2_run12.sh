# round-2 GPU call 12: 3xTF32 GEMM bottleneck experiments (perf-only
# variants: no operand loads after the first ring, no lo*hi MMA, no phase
# folds, both), GPU suite, C3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default noloads nolohi nophase both; do
  if [ $v = default ]; then L=""; else L="--lib paper_2510_10129_b200/variants/libcc_$v.so"; fi
  echo "== $v" >> gpurun_out/r12_gemm.log
  timeout 300 python scripts/bench_gemm.py --only tf32 $L >> gpurun_out/r12_gemm.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r12_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r12_rc.txt
timeout 900 python bench.py > gpurun_out/r12_bench.json 2> gpurun_out/r12_bench.err
echo done
