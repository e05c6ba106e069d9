# round-2 GPU call 54: 3xTF32 GEMMs on CTA pairs (no phases yet) - timing only
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for p in 0 1; do
  echo "== CC_TF32_PAIR=$p rep $rep" >> gpurun_out/r54_gemm.log
  CC_TF32_PAIR=$p timeout 300 python scripts/bench_gemm.py --only tf32x3 >> gpurun_out/r54_gemm.log 2>&1 || CC_TF32_PAIR=$p timeout 300 python scripts/bench_gemm.py >> gpurun_out/r54_gemm.log 2>&1
done
done
cat gpurun_out/r54_gemm.log
