cd $GRAFT_REPO_ROOT
python scripts/profile_run.py --config C2 --max-passes 200 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass_fused -s 1 -c 1 -o gpurun_out/prof_c2_fused python scripts/profile_run.py --config C2 --max-passes 200 > gpurun_out/ncu_c2.log 2>&1
echo rc=$?
