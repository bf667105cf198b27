# quick GPU check: parity tests (fast subset) + C2/C4 bench lines
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_scale" > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2_rc=$?
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --pass-csv gpurun_out/c4_passes.csv > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4_rc=$?
