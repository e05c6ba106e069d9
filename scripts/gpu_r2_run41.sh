# round-2 GPU call 41: banding rule (m fastest only for small A + large B): GEMM tests, C3 bench A/B incl. full prefill
# and chunk precompute (M = 34,816), ncu DRAM of the four recompute GEMMs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm" > gpurun_out/r41_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r41_rc.txt
for rep in 1 2; do
  CC_GEMM_GROUP=0 timeout 900 python bench.py --skip-cpu --no-sweep > gpurun_out/r41_c3_g0_$rep.json 2>/dev/null
  timeout 900 python bench.py --skip-cpu --no-sweep > gpurun_out/r41_c3_new_$rep.json 2>/dev/null
done
ARGS="--steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu --no-sweep"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --nvtx --nvtx-include "timed/" \
  -k regex:"gemm2_kernel" -s 4 -c 4 --csv --log-file gpurun_out/r41_ncu_new.csv python bench.py $ARGS > /dev/null 2>&1
echo done
