cd $GRAFT_REPO_ROOT
MODEL_MODE=p2p timeout 1200 python scripts/exp_scaling_model.py C4 250.6 0.22 2.6595e10 out > gpurun_out/model_p2p_c4_out.txt 2>&1; echo p2p_rc=$?
tail -4 gpurun_out/model_p2p_c4_out.txt | cut -c1-300
MODEL_MODE=async timeout 1200 python scripts/exp_scaling_model.py C4 250.6 0.22 2.6595e10 out > gpurun_out/model_async_c4_out.txt 2>&1; echo async_rc=$?
tail -4 gpurun_out/model_async_c4_out.txt | cut -c1-300
