cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
MODEL_PILOT=0 MODEL_MODE=p2p MODEL_ROUND_PASSES=1 timeout 2400 python scripts/exp_scaling_model.py C3 126.2 0.027 1.669e10 out > gpurun_out/r4_scaling_model_c3_p2p_r1.txt 2>&1; echo rc=$?
grep "^K=" gpurun_out/r4_scaling_model_c3_p2p_r1.txt
MODEL_PILOT=0 MODEL_MODE=async MODEL_ROUND_PASSES=1 timeout 2400 python scripts/exp_scaling_model.py C3 126.2 0.027 1.669e10 out > gpurun_out/r4_scaling_model_c3_async_r1.txt 2>&1; echo rc=$?
grep "^K=" gpurun_out/r4_scaling_model_c3_async_r1.txt
MODEL_PILOT=0 MODEL_MODE=async MODEL_REMOTE_PUSH=0 MODEL_ROUND_PASSES=1 timeout 2400 python scripts/exp_scaling_model.py C3 126.2 0.027 1.669e10 out > gpurun_out/r4_scaling_model_c3_async_r1_perdiff.txt 2>&1; echo rc=$?
grep "^K=" gpurun_out/r4_scaling_model_c3_async_r1_perdiff.txt
