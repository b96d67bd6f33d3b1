# multi-rank code paths on ONE GPU (gloo, host-staged): head-shard bench with
# the per-layer all-gather, and the two-process sequence-shard test (run under gpurun)
cd $GRAFT_REPO_ROOT
[ -n "$SKIP_TESTS" ] || timeout 600 python -m pytest tests/test_gpu_shard_mp.py tests/test_gpu_shard.py -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --workload llama3-8b-32k --dist-backend gloo --no-cpu-baseline --no-full --no-swaps > gpurun_out/mp_bench.txt 2>&1
grep -v "^\s*$" gpurun_out/mp_bench.txt | grep -i "error\|Traceback\|File \"" | head -20; tail -2 gpurun_out/mp_bench.txt
