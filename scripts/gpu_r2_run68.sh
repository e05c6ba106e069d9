# round-2 GPU call 68: bf16 CTA-pair GEMM tile-schedule band A/B on the C3 recompute shapes (isolated)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for g in default 0 4 8 13 26; do
  echo "== band $g rep $rep" >> gpurun_out/r68_band.log
  if [ $g = default ]; then
    timeout 300 python scripts/bench_gemm.py --only bf16 >> gpurun_out/r68_band.log 2>&1
  else
    CC_GEMM_GROUP=$g timeout 300 python scripts/bench_gemm.py --only bf16 >> gpurun_out/r68_band.log 2>&1
  fi
done
done
grep -E "==|bf16 (qkv|o|up|down) " gpurun_out/r68_band.log
