cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/t15.txt 2>&1; tail -3 gpurun_out/t15.txt
