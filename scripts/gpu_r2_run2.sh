# round-2 GPU call 2: scoring precision diagnostic + compute-sanitizer pass
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/diag_scoring_precision.py c2 c3 > gpurun_out/r2_diag.log 2>&1
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider \
    > gpurun_out/r2_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_sanitizer_rc.txt
done
echo done
