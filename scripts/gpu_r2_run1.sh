cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_scale_parity.py -q -s > gpurun_out/r2_scale.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo done
