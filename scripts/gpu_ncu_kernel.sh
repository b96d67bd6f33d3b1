# ncu --set full of one kernel (KREGEX) in a short bench run; report under gpurun_out/
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-2} -c 1 \
  -o gpurun_out/${TAG:-k} python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline --no-swaps ${BENCH_ARGS} > gpurun_out/ncu_${TAG:-k}.log 2>&1
tail -3 gpurun_out/ncu_${TAG:-k}.log
