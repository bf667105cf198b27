cd $GRAFT_REPO_ROOT
python scripts/profile_run.py --config C4 --max-passes 44 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_select" -s 80 -c 2 -o gpurun_out/prof_c4_sparse python scripts/profile_run.py --config C4 --max-passes 44 > gpurun_out/ncu_sparse.log 2>&1
echo rc=$?
