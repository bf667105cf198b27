# Round profile: plain bench, ncu launch list of the same bench command, ncu --set full
# of k_select/k_scatter on a C4 solve (profile_run.py).  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launch_rc=$?
python scripts/profile_run.py --config C4 --max-passes 24 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_select|k_scatter" -s 20 -c 4 -o gpurun_out/prof_c4_full python scripts/profile_run.py --config C4 --max-passes 24 > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
