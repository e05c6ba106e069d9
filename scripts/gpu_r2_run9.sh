# round-2 GPU call 9: work-aware split-KV for small attention grids (low
# ratios, default 8/5 rule, last-layer head row): GPU suite, C3 bench (sweep),
# default-rule launch lists, C2 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r9_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r9_rc.txt
timeout 900 python bench.py > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err
echo "bench rc=$?" >> gpurun_out/r9_rc.txt
timeout 600 python bench.py --config c2 --skip-cpu --no-sweep > gpurun_out/r9_bench_c2.json 2> gpurun_out/r9_bench_c2.err
OUT=r9_launches_dr05 BENCHARGS="--ratio 0.05 --window-threshold 5 --no-sweep" sh scripts/launch_list.sh
OUT=r9_launches_dr20 BENCHARGS="--ratio 0.2 --window-threshold 5 --no-sweep" sh scripts/launch_list.sh
OUT=r9_launches_c3 sh scripts/launch_list.sh
echo done
