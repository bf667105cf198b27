# Scaling model: threshold-coupling floor max_q T_q / alpha^p for p = 2 (build), 1, 0; one pilot solve; new tests again
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_contract.py -q -k "pilot or distributed_path" 2>&1 | tail -3
for v in floor1 floor0; do
  echo "== $v"
  DITER_LIB=$PWD/variants/v_$v.so MODEL_K=2,8 MODEL_PILOT=1 MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 1200 python scripts/exp_scaling_model.py C4 176.5 0.072 2.306e10 out 2>&1 | grep "^K="
done 2>&1 | tee gpurun_out/r4_model_floor.txt
echo "== round passes 1 (floor pow 2)" | tee -a gpurun_out/r4_model_floor.txt
MODEL_K=2,8 MODEL_PILOT=1 MODEL_MODE=p2p MODEL_ROUND_PASSES=1 timeout 1200 python scripts/exp_scaling_model.py C4 176.5 0.072 2.306e10 out 2>&1 | grep "^K=" | tee -a gpurun_out/r4_model_floor.txt
