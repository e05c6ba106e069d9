# round-2 GPU call 67: compute-sanitizer on the 3xTF32 CTA-pair GEMM tests (sanitizer build, see profiles/r2_sanitizer.md)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CACHECLIP_SM100_LIB=paper_2510_10129_b200/variants/libcc_sanitize.so
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "tf32" \
    > gpurun_out/r67_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r67_rc.txt
  tail -n 4 gpurun_out/r67_sanitizer_$tool.log >> gpurun_out/r67_rc.txt
done
cat gpurun_out/r67_rc.txt
