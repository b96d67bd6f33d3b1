# quick iteration loop on the GPU box: parity tests, step timeline, short bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/pytest.txt
tail -5 gpurun_out/pytest.txt
timeout 300 python scripts/step_timeline.py > gpurun_out/timeline.txt 2>&1
tail -12 gpurun_out/timeline.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -3 gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print("value us/token", round(d["value"], 1), "frac", round(d["roofline"]["frac"], 3),
      "full", d["full_attention"] and round(d["full_attention"]["us_per_token"], 1),
      "speedup", d["full_attention"] and round(d["full_attention"]["speedup_hybrid_vs_full"], 3),
      "e2e", round(d["e2e"]["value"], 1), "clk", d["clocks"])
PY
