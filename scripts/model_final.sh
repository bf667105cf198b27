cd $GRAFT_REPO_ROOT
MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 1200 python scripts/exp_scaling_model.py C4 248.8 0.224 2.6595e10 out > gpurun_out/r02_scaling_model_c4_p2p.txt 2>&1; echo p2p=$?
grep "^K=" gpurun_out/r02_scaling_model_c*.txt
