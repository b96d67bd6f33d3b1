# A/B of the working build against liblyc_base.so (run under gpurun):
# selection phases + short bench for both, interleaved twice
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in base new; do
  if [ $v = base ]; then export LYC_LIB_VARIANT=base; else unset LYC_LIB_VARIANT; fi
  echo "== $v (round $r)"
  timeout 300 python scripts/sel_phases.py 2>&1 | tail -13
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
done
