cd ${GRAFT_REPO_ROOT:-.}
export DITER_LIB=$PWD/variants/v_win2.so
ncu --set full --clock-control none --import-source on -k regex:k_sweep_win --launch-skip 5 --launch-count 1 -o gpurun_out/r3_win2_c4 -f \
  python scripts/profile_run.py --config C4 --max-passes 8 --opt sweep=2 --opt scatter_run=16 > gpurun_out/ncu_win.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/ncu_win.log
