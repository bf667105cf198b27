# ncu --set full of two mid-solve C2 passes (select + scatter), L2 left warm between
# replays (C2's working set is L2-resident in the real run)
cd $GRAFT_REPO_ROOT
python scripts/profile_run.py --config C2 --max-passes 400 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k_scatter|k_select" -s 60 -c 4 \
    -o gpurun_out/prof_c2_r01 python scripts/profile_run.py --config C2 --max-passes 400 > gpurun_out/ncu_run.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_run.log
