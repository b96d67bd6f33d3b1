# round-2 evidence: launch list + ncu --set full of the step kernel (qwen3-8b-128k)
# and of the tcgen05 window kernel (run under gpurun)
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline --no-swaps --no-model --no-sweep --no-flashinfer > /dev/null 2>&1
echo "launch rows: $(wc -l < gpurun_out/r2_launches.csv)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hybrid_step -s 3 -c 1 \
  -o gpurun_out/r2_step python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline --no-swaps --no-model --no-sweep --no-flashinfer > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:window_tc_kernel -s 3 -c 1 \
  -o gpurun_out/r2_window python scripts/bench_window.py > gpurun_out/ncu_window.log 2>&1
tail -2 gpurun_out/ncu_window.log
