# round-2 GPU call 6 (after container re-create): full GPU suite, smoke, C3 bench, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r6_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r6_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r6_bench.json 2> gpurun_out/r6_bench.err
OUT=r6_launches sh scripts/launch_list.sh
echo done
