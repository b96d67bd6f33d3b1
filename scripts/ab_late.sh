cd $GRAFT_REPO_ROOT
for v in base new; do
  if [ $v = base ]; then export LYC_LIB_VARIANT=base; else unset LYC_LIB_VARIANT; fi
  echo "== $v"
  timeout 300 python scripts/cta_late.py 2>&1 | head -32 | awk '{print $1,$2,$4,$5,$6,$7,$9,$10,$11,$12}' | head -32 > /tmp/late_$v.txt
  python - <<'PY'
import re,sys
PY
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
paste /tmp/late_base.txt /tmp/late_new.txt | head -32
