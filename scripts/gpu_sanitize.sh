# compute-sanitizer over the round-2 kernels (run under gpurun)
cd $GRAFT_REPO_ROOT
for t in "tests/test_gpu_kvcache.py" "tests/test_gpu_model.py" "tests/test_gpu_decode.py -k tiny_config"; do
  timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest $t -q -x -p no:cacheprovider > gpurun_out/san.log 2>&1
  echo "memcheck [$t] rc=$? $(grep -c 'Invalid\|ERROR SUMMARY' gpurun_out/san.log) $(grep 'ERROR SUMMARY' gpurun_out/san.log | tail -1) $(tail -1 gpurun_out/san.log)"
done
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_kvcache.py -q -x -p no:cacheprovider > gpurun_out/san2.log 2>&1
echo "synccheck kvcache rc=$? $(grep 'ERROR SUMMARY' gpurun_out/san2.log | tail -1) $(tail -1 gpurun_out/san2.log)"
