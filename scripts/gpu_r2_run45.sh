# round-2 GPU call 45: host-side profile of a C3 request (exact-budget and default rule); timeline after the
# merged token-id fix
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/dbg_host_prof.py 1 > gpurun_out/r45_host1.log 2>&1
timeout 300 python scripts/dbg_host_prof.py 5 > gpurun_out/r45_host5.log 2>&1
timeout 300 python scripts/dbg_timeline.py c3 0.2 5 > gpurun_out/r45_timeline.log 2>&1
timeout 300 python scripts/dbg_timeline.py c3 0.2 1 >> gpurun_out/r45_timeline.log 2>&1
echo done
