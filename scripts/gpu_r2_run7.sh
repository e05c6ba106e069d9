# round-2 GPU call 7 (session 3, container re-created): GPU suite, smoke, C3 bench,
# launch list, compute-sanitizer memcheck/racecheck/synccheck on kernel + sharded tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r7_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r7_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r7_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r7_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r7_rc.txt
timeout 900 python bench.py > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err
echo "bench rc=$?" >> gpurun_out/r7_rc.txt
export CACHECLIP_SM100_LIB=paper_2510_10129_b200/variants/libcc_sanitize.so
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py tests/test_gpu_api.py -q -p no:cacheprovider -k "not fullsize" \
    > gpurun_out/r7_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r7_rc.txt
done
echo done
