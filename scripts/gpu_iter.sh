# quick iteration loop on the GPU box: new-path tests, full GPU suite, timeline, bench
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_plan.py -q -x -p no:cacheprovider > gpurun_out/pytest_plan.txt 2>&1
tail -15 gpurun_out/pytest_plan.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/step_timeline.py --workload qwen3-8b-128k --save gpurun_out/trace.npy > gpurun_out/timeline.txt 2>&1
tail -3 gpurun_out/timeline.txt
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -3 gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print("value us/token", round(d["value"], 1), "frac", round(d["roofline"]["frac"], 3),
      "full", d["full_attention"] and round(d["full_attention"]["us_per_token"], 1),
      "speedup", d["full_attention"] and round(d["full_attention"]["speedup_hybrid_vs_full"], 3),
      "e2e", d["e2e"], "per_layer", d["per_layer_api"], "swaps", d["selection_swaps"], "clk", d["clocks"])
PY
