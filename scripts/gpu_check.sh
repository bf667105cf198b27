# quick GPU check: every -m gpu test except the full-scale ones
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -k "not full_scale and not 2_31 and not max_nodes" > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/gpu_tests.log
