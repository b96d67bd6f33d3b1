# A/B: the current build vs an older worktree build (build/r2a), same box, alternating
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for v in new old; do
    if [ $v = new ]; then D=.; X="--no-swaps $NEWARGS"; else D=build/r2a; X=""; fi
    (cd $D && timeout 600 python bench.py --workload qwen3-8b-128k --steps 30 --warmup 5 --no-cpu-baseline --no-full $X 2>/dev/null) | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'value', round(d['value'],1), 'kernel_us', round(d['roofline']['attn_us_per_step'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done
