# round-2 GPU call 3: phased 3xTF32 accumulation -> precision diag, kernel +
# scale parity tests, sanitizer (racecheck/synccheck) on the sync-load variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" -s > gpurun_out/r3_gemm.log 2>&1
timeout 900 python scripts/diag_scoring_precision.py c2 c3 > gpurun_out/r3_diag.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -s > gpurun_out/r3_scale.log 2>&1
export CACHECLIP_SM100_LIB=paper_2510_10129_b200/variants/libcc_sanitize.so
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py -q -p no:cacheprovider \
    > gpurun_out/r3_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r3_sanitizer_rc.txt
done
echo done
