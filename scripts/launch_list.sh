# per-launch device times of one timed bench step (ncu, serialised launches); run under gpurun
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
  --csv --log-file gpurun_out/${OUT:-launches}.csv python bench.py --steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu ${BENCHARGS:-} \
  > gpurun_out/${OUT:-launches}.log 2>&1
tail -2 gpurun_out/${OUT:-launches}.log
