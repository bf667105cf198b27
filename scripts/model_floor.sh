cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ipc.py -q --timeout 600 -k "p2p" > gpurun_out/gpu_p2p.log 2>&1; echo p2p_rc=$?; tail -2 gpurun_out/gpu_p2p.log
echo floor C4; MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 1200 python scripts/exp_scaling_model.py C4 248.8 0.224 2.6595e10 out 2>&1 | grep "^K="
echo nofloor C4; DITER_LIB=$PWD/variants/v_nofloor.so MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 1200 python scripts/exp_scaling_model.py C4 248.8 0.224 2.6595e10 out 2>&1 | grep "^K="
echo floor C3; MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 1200 python scripts/exp_scaling_model.py C3 181.4 0.129 1.8700e10 out 2>&1 | grep "^K="
echo floor4 C4; MODEL_MODE=p2p MODEL_ROUND_PASSES=4 timeout 1200 python scripts/exp_scaling_model.py C4 248.8 0.224 2.6595e10 out 2>&1 | grep "^K="
