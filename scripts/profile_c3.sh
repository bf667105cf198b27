# C3 (R-MAT 2^24) profile in bench's launch configuration: ncu launch list of the bench
# command, then --set full of one mid-solve pass (select, scatter, hubs).
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/c3_plain.json 2> gpurun_out/c3_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_c3_launch.log 2>&1
echo launch_rc=$?
timeout 300 python scripts/profile_run.py --config C3 --max-passes 64 > gpurun_out/c3_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select|k_scatter" -s 120 -c 3 -o gpurun_out/prof_c3_full python scripts/profile_run.py --config C3 --max-passes 64 > gpurun_out/ncu_c3_full.log 2>&1
echo full_rc=$?
