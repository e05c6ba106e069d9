# round-2 GPU call 5: GPU suite, GEMM microbench (3xTF32 phase length variants,
# fused-norm epilogues), precision diag at P=8, C3 bench, sanitizer (attention)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/r5_gpu.log 2>&1
for v in default p2 p8 p1000; do
  if [ $v = default ]; then L=""; else L="--lib paper_2510_10129_b200/variants/libcc_$v.so"; fi
  echo "== $v" >> gpurun_out/r5_gemm.log
  timeout 300 python scripts/bench_gemm.py $L >> gpurun_out/r5_gemm.log 2>&1
done
CACHECLIP_SM100_LIB=paper_2510_10129_b200/variants/libcc_p8.so timeout 600 python scripts/diag_scoring_precision.py c3 > gpurun_out/r5_diag_p8.log 2>&1
cp gpurun_out/diag_scoring_c3.json gpurun_out/r5_diag_p8_c3.json
timeout 900 python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
export CACHECLIP_SM100_LIB=paper_2510_10129_b200/variants/libcc_sanitize.so
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py -q -p no:cacheprovider -k "attention" \
    > gpurun_out/r5_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r5_sanitizer_rc.txt
done
echo done
