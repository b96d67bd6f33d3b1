# A/B of library builds (run under gpurun): every build/variants/<name>/liblyc.so
# is swapped in for paper_2602_04541_b200/liblyc.so in turn, interleaved
# ROUNDS times, and one bench case per WORKLOADS entry is run with it.
cd $GRAFT_REPO_ROOT
cp paper_2602_04541_b200/liblyc.so build/liblyc_keep.so
for r in $(seq 1 ${ROUNDS:-2}); do
for v in build/variants/*/; do
  n=$(basename $v)
  cp $v/liblyc.so paper_2602_04541_b200/liblyc.so
  for w in ${WORKLOADS:-qwen3-8b-128k}; do
    timeout 300 python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --no-full --no-swaps \
      --no-model --no-flashinfer --no-sweep --workload $w $ARGS 2>gpurun_out/var_err.txt | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
    print('[$n r$r $w]', 'value', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'per_layer_graph', d['per_layer_api'] and round(d['per_layer_api']['us_per_token_graph'],1))
except Exception as e:
    print('[$n r$r $w] FAILED', e); print(open('gpurun_out/var_err.txt').read()[-1500:])"
  done
done
done
cp build/liblyc_keep.so paper_2602_04541_b200/liblyc.so
