# ncu --set full of one kernel (regex $K, skip $SKIP launches) inside bench's timed range; run under gpurun
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu ${BENCHARGS:-}"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
  --kernel-name-base mangled -k regex:"$K" -s ${SKIP:-0} -c 1 -o gpurun_out/$OUT python bench.py $ARGS > gpurun_out/$OUT.log 2>&1
tail -3 gpurun_out/$OUT.log
