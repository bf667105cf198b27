# quick GPU check: parity tests (fast subset) + C2/C4 bench lines
cd $GRAFT_REPO_ROOT
free -g | head -2; nproc
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -k "not full_scale and not 2_31 and not max_nodes" > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2_rc=$?
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-raw-key --pass-csv gpurun_out/c4_passes.csv > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4_rc=$?
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
