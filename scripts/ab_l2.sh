# A/B of variants x L2 window sizes on C4/C3:  bash scripts/ab_l2.sh "base hint" "0 32 48"
cd ${GRAFT_REPO_ROOT:-.}
VARIANTS=${1:-"base hint"}; WINS=${2:-"0"}; CONFIGS=${3:-"C4 C3"}
for c in $CONFIGS; do for w in $WINS; do for v in $VARIANTS; do
  echo "$c $v l2=$w $(DITER_LIB=$PWD/variants/v_$v.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-raw-key --l2-persist $w 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],3), round(r['kernel_shares']['k_scatter'],3), round(r['frac'],4))")"
done; done; done
