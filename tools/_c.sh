cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_guards.py tests/test_gpu_dist.py -q > gpurun_out/t14.txt 2>&1; tail -3 gpurun_out/t14.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k async > gpurun_out/t14b.txt 2>&1; tail -2 gpurun_out/t14b.txt
