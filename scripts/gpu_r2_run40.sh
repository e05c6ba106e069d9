# round-2 GPU call 40: banded persistent schedule for the CTA-pair GEMM (down projection):
# bitwise test, GEMM-alone A/B over the band size, C3 bench A/B, ncu DRAM bytes of the down GEMM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm" > gpurun_out/r40_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r40_rc.txt
for rep in 1 2; do
for g in 0 4 8 12; do
  echo "== CC_GEMM_GROUP=$g" >> gpurun_out/r40_gemm.log
  CC_GEMM_GROUP=$g timeout 300 python scripts/bench_gemm.py >> gpurun_out/r40_gemm.log 2>&1
done
done
for rep in 1 2; do
  CC_GEMM_GROUP=0 timeout 600 python bench.py --skip-cpu --skip-full --no-sweep > gpurun_out/r40_c3_g0_$rep.json 2>/dev/null
  timeout 600 python bench.py --skip-cpu --skip-full --no-sweep > gpurun_out/r40_c3_g8_$rep.json 2>/dev/null
done
ARGS="--steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu --no-sweep"
for g in 0 8; do
CC_GEMM_GROUP=$g timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --nvtx --nvtx-include "timed/" \
  -k regex:"gemm2_kernel" -s 4 -c 4 --csv --log-file gpurun_out/r40_ncu_g$g.csv python bench.py $ARGS > /dev/null 2>&1
done
echo done
