# round-2 GPU call 11: vectorised LSE merge; ncu --set full of the 3xTF32 up
# and down GEMMs (scoring pass); default-rule launch list; decode
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py tests/test_gpu_api.py -q -x -p no:cacheprovider > gpurun_out/r11_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r11_rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 4 \
  -o gpurun_out/r11_tf32 python scripts/bench_gemm.py --only tf32 --reps 1 --trials 1 > gpurun_out/r11_tf32_ncu.log 2>&1
OUT=r11_launches_dr05 BENCHARGS="--ratio 0.05 --window-threshold 5 --no-sweep" sh scripts/launch_list.sh
timeout 600 python scripts/bench_decode.py > gpurun_out/r11_decode.log 2>&1
echo done
