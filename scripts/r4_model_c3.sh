# Scaling model for C3 (permuted R-MAT) with sweeps on every rank, performed-push accounting
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
MODEL_PILOT=0 MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 2400 python scripts/exp_scaling_model.py C3 126.2 0.027 1.669e10 out > gpurun_out/r4_scaling_model_c3_p2p.txt 2>&1; echo rc=$?
grep "^K=" gpurun_out/r4_scaling_model_c3_p2p.txt
MODEL_PILOT=0 MODEL_MODE=p2p MODEL_ROUND_PASSES=4 timeout 2400 python scripts/exp_scaling_model.py C3 126.2 0.027 1.669e10 out > gpurun_out/r4_scaling_model_c3_p2p_r4.txt 2>&1; echo rc=$?
grep "^K=" gpurun_out/r4_scaling_model_c3_p2p_r4.txt
