# round-2 GPU call 60: C2 / C5 / C4 (sharded W=1) bench lines at HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config c2 --skip-cpu > gpurun_out/r60_bench_c2.json 2> gpurun_out/r60_bench_c2.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/r60_bench_c5.json 2> gpurun_out/r60_bench_c5.err
timeout 1500 python bench.py --config c4 --sharded --steps 2 --warmup 1 > gpurun_out/r60_bench_c4.json 2> gpurun_out/r60_bench_c4.err
for f in c2 c5 c4; do head -c 300 gpurun_out/r60_bench_$f.json; echo; tail -n 2 gpurun_out/r60_bench_$f.err; done
