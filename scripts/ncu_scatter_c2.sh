cd $GRAFT_REPO_ROOT
python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_scatter -s 20 -c 2 -o gpurun_out/prof_c2_scatter python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_run.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_run.log
