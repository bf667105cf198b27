# Scaling model (loopback ranks on one GPU) with pilot-measured re-balancing of the ranges
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
MODEL_PILOT=2 MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 2400 python scripts/exp_scaling_model.py C4 176.5 0.072 2.306e10 out > gpurun_out/r4_scaling_model_c4_p2p_pilot2.txt 2>&1; echo rc=$?
grep "^K=" gpurun_out/r4_scaling_model_c4_p2p_pilot2.txt
