# round-2 GPU call 39: scoring pass in-request vs alone (per-launch profiler); launch list and
# ncu --set full of the attention kernel (layer 3) with the P parts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/dbg_scoring_prof.py > gpurun_out/r39_scoring.log 2>&1
ARGS="--steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
  --csv --log-file gpurun_out/r39_launches_c3.csv python bench.py $ARGS > gpurun_out/r39_launches_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" --kernel-name-base mangled \
  -k regex:"fa_sparse_row" -s 3 -c 1 -o gpurun_out/r39_prof_fa python bench.py $ARGS > gpurun_out/r39_prof_fa.log 2>&1
echo done
