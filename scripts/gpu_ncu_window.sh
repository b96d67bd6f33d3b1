# ncu --set full of the tensor-core window attention kernel (run under gpurun)
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:window_tc_kernel -s 3 -c 1 \
  -o gpurun_out/window_tc python scripts/bench_window.py > gpurun_out/ncu_window.log 2>&1
tail -3 gpurun_out/ncu_window.log
