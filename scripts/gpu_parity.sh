# BASELINE-size parity tests + the full GPU suite (run under gpurun)
cd $GRAFT_REPO_ROOT
export LYC_PARITY_REPORT=gpurun_out/parity_report.jsonl
rm -f $LYC_PARITY_REPORT
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -s -x -p no:cacheprovider > gpurun_out/parity.txt 2>&1
tail -25 gpurun_out/parity.txt
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.txt 2>&1
tail -6 gpurun_out/pytest_gpu.txt
