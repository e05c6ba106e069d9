# round-2 GPU call 4: full GPU suite (fused RMSNorm, phased 3xTF32, multi-process
# sharded), C3 bench, sanitizer (no setmaxnreg) on the attention tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/r4_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err
export CACHECLIP_SM100_LIB=paper_2510_10129_b200/variants/libcc_sanitize.so
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py -q -p no:cacheprovider -k "attention" \
    > gpurun_out/r4_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r4_sanitizer_rc.txt
done
echo done
