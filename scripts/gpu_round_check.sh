set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1s9_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s9_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r1s9_bench.json 2> gpurun_out/r1s9_bench.err
tail -3 gpurun_out/r1s9_gpu_tests.log; cat gpurun_out/r1s9_smoke.log | tail -3; cat gpurun_out/r1s9_bench.json; tail -5 gpurun_out/r1s9_bench.err
