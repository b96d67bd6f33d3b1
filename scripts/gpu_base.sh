cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
timeout 300 python scripts/step_timeline.py --workload qwen3-8b-128k --save gpurun_out/r2_base_trace.npy > gpurun_out/r2_base_timeline.txt 2>&1
tail -40 gpurun_out/r2_base_timeline.txt
timeout 600 python bench.py --workload qwen3-8b-128k --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err
tail -3 gpurun_out/r2_base_bench.err; tail -c 1500 gpurun_out/r2_base_bench.json
