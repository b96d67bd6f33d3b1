# bench + ncu evidence for the current build (run under gpurun)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r1}
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline > /dev/null 2>&1
echo "launch list rows: $(wc -l < gpurun_out/launches_$TAG.csv)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hybrid_attn -s 32 -c 2 \
  -o gpurun_out/attn_$TAG python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline > gpurun_out/ncu_attn_$TAG.log 2>&1
tail -3 gpurun_out/ncu_attn_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk -s 4 -c 1 \
  -o gpurun_out/topk_$TAG python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline > gpurun_out/ncu_topk_$TAG.log 2>&1
tail -2 gpurun_out/ncu_topk_$TAG.log
