# per-kernel durations of the first passes of a C4 solve (args: extra profile_run options)
cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_far.csv python scripts/profile_run.py --config C4 --max-passes 6 "$@" > gpurun_out/ncu_launch_far.log 2>&1
echo rc=$?
