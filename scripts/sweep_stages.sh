# ring-depth sweep of the fused step (bench value, no full-attention / CPU legs)
cd $GRAFT_REPO_ROOT
for st in 2 3 4; do
  echo "== LYC_STAGES=$st"
  LYC_STAGES=$st timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1))"
done
