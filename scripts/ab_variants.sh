# A/B of library builds under variants/ (scripts/build_variant.py) through bench.py:
#   bash scripts/ab_variants.sh "C4 C3" "base tp" [reps]
cd ${GRAFT_REPO_ROOT:-.}
CONFIGS=${1:-"C4 C3"}; VARIANTS=${2:-"base tp"}; REPS=${3:-2}
for c in $CONFIGS; do for r in $(seq $REPS); do for v in $VARIANTS; do
  echo "$c $v $(DITER_LIB=$PWD/variants/v_$v.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_shares']['k_scatter'],3), round(d['roofline']['atomic_issue']['frac'],3))")"
done; done; done
