# Scaling model: relative sleep rule (options.p2p_sleep = k %) with one pilot solve
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for k in 10 30 60; do
  echo "== p2p_sleep $k"
  MODEL_SLEEP=$k MODEL_K=2,8 MODEL_PILOT=1 MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 900 python scripts/exp_scaling_model.py C4 176.5 0.072 2.306e10 out 2>&1 | grep "^K=\|Error\|error"
done 2>&1 | tee gpurun_out/r4_model_sleep.txt
