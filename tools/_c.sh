cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/t11.txt 2>&1; tail -3 gpurun_out/t11.txt
