# ncu --set full of k_select/k_scatter at C4 passes 10-12 (pass 10 dense ~26 %, 12 sparse ~5 %)
cd $GRAFT_REPO_ROOT
python scripts/profile_run.py --config C4 --max-passes 24 > gpurun_out/plain_p10.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_select|k_scatter" -s 20 -c 6 -o gpurun_out/prof_c4_p10 python scripts/profile_run.py --config C4 --max-passes 24 > gpurun_out/ncu_p10.log 2>&1
echo rc=$?
