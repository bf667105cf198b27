cd $GRAFT_REPO_ROOT
for c in in/4 in/8 in/16; do echo "p2p round2 $c"; MODEL_K=8 MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 1200 python scripts/exp_scaling_model.py C4 248.8 0.224 2.6595e10 $c > gpurun_out/mp_$(echo $c | tr / _).txt 2>&1; grep "^K=" gpurun_out/mp_$(echo $c | tr / _).txt; done
