# run bench.py once per argument set in CASES (separated by ';') and print
# the headline numbers (run under gpurun)
cd $GRAFT_REPO_ROOT
IFS=';' read -ra CS <<< "$CASES"
for c in "${CS[@]}"; do
  timeout 600 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-full --no-swaps --no-sweep ${EXTRA:---no-model} $c 2>gpurun_out/case_err.txt | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read().strip().splitlines()[-1])
    pl=d['per_layer_api']
    print('[$c]', 'value', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'bytes', round(d['roofline']['bytes_per_step']/1e9,3), 'e2e', round(d['e2e']['value'],1), 'per_layer_graph', pl and round(pl['us_per_token_graph'],1), 'model', d.get('model_tpot'))
except Exception as e:
    print('[$c] FAILED', e); print(open('gpurun_out/case_err.txt').read()[-1500:])"
done
