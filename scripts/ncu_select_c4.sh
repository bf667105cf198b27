cd $GRAFT_REPO_ROOT
python scripts/profile_run.py --config C4 --max-passes 24 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_select|k_scatter" -s 20 -c 4 -o gpurun_out/prof_c4 python scripts/profile_run.py --config C4 --max-passes 24 > gpurun_out/ncu_run.log 2>&1
echo ncu_rc=$?; tail -2 gpurun_out/ncu_run.log; cat gpurun_out/plain.log
