cd $GRAFT_REPO_ROOT
timeout 300 python scripts/step_timeline.py > gpurun_out/tl_base.txt 2>&1
LYC_NO_HIST16=1 timeout 300 python scripts/step_timeline.py > gpurun_out/tl_nohist16.txt 2>&1
head -6 gpurun_out/tl_base.txt; head -6 gpurun_out/tl_nohist16.txt; tail -1 gpurun_out/tl_base.txt; tail -1 gpurun_out/tl_nohist16.txt
