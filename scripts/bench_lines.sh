cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_c4_reference.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
for c in C2 C3 C5; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo ${c}_rc=$?; done
