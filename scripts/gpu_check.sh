# GPU correctness gate + quick bench (run under gpurun)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest.txt
cat gpurun_out/pytest.txt | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -3 gpurun_out/bench_q.err; cat gpurun_out/bench_q.json
