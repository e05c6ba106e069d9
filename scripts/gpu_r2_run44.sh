# round-2 GPU call 44: launch timeline of a C3 request (idle gaps between launches)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/dbg_timeline.py c3 0.2 1 > gpurun_out/r44_timeline.log 2>&1
timeout 300 python scripts/dbg_timeline.py c3 0.2 5 >> gpurun_out/r44_timeline.log 2>&1
timeout 300 python scripts/dbg_prof_overhead.py > gpurun_out/r44_prof_overhead.log 2>&1
echo done
