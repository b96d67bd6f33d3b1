# bench value of several in-tree library variants (liblyc_<name>.so), interleaved twice
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in ${VARIANTS:-base}; do
  if [ $v = new ]; then unset LYC_LIB_VARIANT; else export LYC_LIB_VARIANT=$v; fi
  echo "== $v $(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))")"
done; done
