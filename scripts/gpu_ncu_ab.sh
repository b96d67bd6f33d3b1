# ncu --set full of the step kernel for the current build and build/r2a
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hybrid_step -s 3 -c 1 -o gpurun_out/step_new python bench.py --steps 2 --warmup 3 --no-full --no-cpu-baseline --no-swaps > gpurun_out/ncu_new.log 2>&1
(cd build/r2a && timeout 900 ncu --set full --clock-control none --import-source on -k regex:hybrid_step -s 3 -c 1 -o ../../gpurun_out/step_old python bench.py --workload qwen3-8b-128k --steps 2 --warmup 3 --no-full --no-cpu-baseline > ../../gpurun_out/ncu_old.log 2>&1)
tail -2 gpurun_out/ncu_new.log gpurun_out/ncu_old.log
