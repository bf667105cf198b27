# Round-2 measurements on one B200: new tests, bench lines of every config (C4 with the
# driver's command), the reference arm, the ncu launch list of the C4 bench command and
# --set full captures of k_scatter on C4 (passes 6-7) and C3 (one mid-solve pass).
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -k "create_failure or needs_default_pagerank" > gpurun_out/new_tests.log 2>&1; echo new_tests_rc=$?; tail -2 gpurun_out/new_tests.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo c4_rc=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_c4_reference.json 2> gpurun_out/r02_ref.err; echo ref_rc=$?
for C in C3 C2 C5 C1; do
  python bench.py --config $C --steps 10 --warmup 3 > gpurun_out/r02_bench_$(echo $C | tr C c).json 2> gpurun_out/r02_bench_$C.err; echo ${C}_rc=$?
done
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-raw-key"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
timeout 300 python scripts/profile_run.py --config C4 --max-passes 10 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_select" -s 12 -c 4 -o gpurun_out/r02_c4_full python scripts/profile_run.py --config C4 --max-passes 10 > gpurun_out/ncu_full_c4.log 2>&1; echo full_c4_rc=$?
timeout 300 python scripts/profile_run.py --config C3 --max-passes 60 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 100 -c 3 -o gpurun_out/r02_c3_full python scripts/profile_run.py --config C3 --max-passes 60 > gpurun_out/ncu_full_c3.log 2>&1; echo full_c3_rc=$?
