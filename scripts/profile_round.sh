# Round profile (C4, bench launch configuration): plain bench line, ncu launch list of
# the same bench command, ncu --set full of k_select/k_scatter at a dense and a
# sparse pass (passes 6-7 of profile_run.py).  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launch_rc=$?
timeout 300 python scripts/profile_run.py --config C4 --max-passes 16 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select|k_scatter" -s 12 -c 6 -o gpurun_out/prof_c4_full python scripts/profile_run.py --config C4 --max-passes 16 > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
