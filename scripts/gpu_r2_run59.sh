# round-2 GPU call 59: evidence set at HEAD (launch list + ncu --set full of the top kernels)
cd $GRAFT_REPO_ROOT
bash scripts/profile_r2.sh > gpurun_out/r59_profile.log 2>&1
python scripts/launch_table.py gpurun_out/r2_launches_c3.csv > gpurun_out/r59_launches.txt 2>&1
python scripts/ncu_summary.py gpurun_out/r2_prof_*.ncu-rep > gpurun_out/r59_ncu_full.txt 2>&1
cat gpurun_out/r59_ncu_full.txt | head -5
rm -f gpurun_out/*.ncu-rep gpurun_out/r2_launches_c3.csv
