# everything: GPU suite incl. BASELINE-size parity, timeline, bench (run under gpurun)
cd $GRAFT_REPO_ROOT
export LYC_PARITY_REPORT=gpurun_out/parity_report.jsonl
rm -f $LYC_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -4 gpurun_out/pytest_gpu.txt; cat $LYC_PARITY_REPORT
timeout 300 python scripts/step_timeline.py --workload qwen3-8b-128k --save gpurun_out/trace.npy > gpurun_out/timeline.txt 2>&1
tail -1 gpurun_out/timeline.txt
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -3 gpurun_out/bench_full.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_full.json").read().strip().splitlines()[-1])
print(json.dumps({k: d[k] for k in ("value", "e2e", "per_layer_api", "selection_swaps", "full_attention", "cpu_baseline", "gpu_launches", "clocks")})[:3000])
print("frac", d["roofline"]["frac"])
PY
