cd ${GRAFT_REPO_ROOT:-.}
ncu --metrics gpu__time_duration.sum -k regex:k_sweep --clock-control none --csv --log-file gpurun_out/r3_pc_base.csv \
  python scripts/profile_run.py --config C4 --max-passes 1000 --pass-csv gpurun_out/r3_pc_base_passes.csv > /dev/null 2>&1; echo rc=$?
DITER_LIB=$PWD/variants/v_win2.so ncu --metrics gpu__time_duration.sum -k regex:k_sweep --clock-control none --csv --log-file gpurun_out/r3_pc_win.csv \
  python scripts/profile_run.py --config C4 --max-passes 1000 --opt sweep=2 --opt scatter_run=16 --pass-csv gpurun_out/r3_pc_win_passes.csv > /dev/null 2>&1; echo rc=$?
