cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ipc.py -q --timeout 600 -k "p2p" > gpurun_out/gpu_p2p.log 2>&1; echo p2p_rc=$?; tail -2 gpurun_out/gpu_p2p.log
for v in "1 2.0 0.5" "2 2.0 0.5" "4 2.0 0.5" "8 2.0 0.5"; do set -- $v
  echo "round=$1 alpha=$2 f=$3"
  MODEL_K=8 MODEL_MODE=p2p MODEL_ROUND_PASSES=$1 MODEL_ALPHA=$2 MODEL_FRAC=$3 timeout 600 python scripts/exp_scaling_model.py C4 250.6 0.22 2.6595e10 out 2>&1 | grep "^K="
done
