# round-2 GPU call 63: ncu --set full with source of one context-layer banked scoring attention launch (C3 step)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" --kernel-name-base mangled \
  -k regex:banked_tc -s 3 -c 1 -o gpurun_out/r63_banked python bench.py --steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu --no-sweep > gpurun_out/r63.log 2>&1
ls -la gpurun_out/r63_banked.ncu-rep; tail -n 2 gpurun_out/r63.log
