# A/B of bench variants on one box (BENCH_A / BENCH_B extra args), then the plan-path tests
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_plan.py tests/test_gpu_decode.py -q -x -p no:cacheprovider > gpurun_out/pytest_ab.txt 2>&1
tail -3 gpurun_out/pytest_ab.txt
for v in A B A B; do
  if [ $v = A ]; then X="$BENCH_A"; else X="$BENCH_B"; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-full --no-swaps $X 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$X', 'value', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'kernel_us', round(d['roofline']['attn_us_per_step'],1), 'e2e', round(d['e2e']['value'],1), 'per_layer_graph', d['per_layer_api'] and round(d['per_layer_api']['us_per_token_graph'],1))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"plan_kernel|hybrid_step" -c 8 --log-file gpurun_out/plan_launches.csv python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline --no-swaps > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/plan_launches.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
print([ (r[ki][:12], r[vi]) for r in rows[1:]])
PY
