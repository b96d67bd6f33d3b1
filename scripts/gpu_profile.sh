# bench line + ncu evidence for the current build (run under gpurun)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r1}
WL=${WL:-llama3-8b-128k}
timeout 900 python bench.py --workload $WL --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --workload $WL --steps 2 --warmup 3 --no-full --no-cpu-baseline > /dev/null 2>&1
echo "launch list rows: $(wc -l < gpurun_out/launches_$TAG.csv)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hybrid_step -s 3 -c 1 \
  -o gpurun_out/step_$TAG python bench.py --workload $WL --steps 2 --warmup 3 --no-full --no-cpu-baseline > gpurun_out/ncu_step_$TAG.log 2>&1
tail -2 gpurun_out/ncu_step_$TAG.log
