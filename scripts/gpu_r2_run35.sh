# round-2 GPU call 35: P handed to the PV MMA in parts (CC_FA_PV_PARTS 1/2/4):
# attention alone on the C3 recompute shape, the per-tile timeline, attention tests, C3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for lib in paper_2510_10129_b200/variants/libcc_pv1.so paper_2510_10129_b200/libcacheclip_sm100.so paper_2510_10129_b200/variants/libcc_pv4.so; do
  timeout 120 python scripts/bench_attention.py --lib $lib --dense 32768 >> gpurun_out/r35_attn.log 2>&1
done
done
timeout 120 python scripts/dbg_fa_trace.py paper_2510_10129_b200/variants/libcc_trace1.so > gpurun_out/r35_trace1.log 2>&1
timeout 120 python scripts/dbg_fa_trace.py paper_2510_10129_b200/variants/libcc_trace.so > gpurun_out/r35_trace2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "attention or attn" > gpurun_out/r35_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r35_rc.txt
timeout 600 python bench.py --skip-cpu > gpurun_out/r35_bench_c3.json 2> gpurun_out/r35_bench_c3.err
echo "c3 rc=$?" >> gpurun_out/r35_rc.txt
echo done
