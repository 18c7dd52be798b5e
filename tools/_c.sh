cd $GRAFT_REPO_ROOT
python tools/ab_lib.py paper_2006_07583_b200/ab/cur2.so,paper_2006_07583_b200/ab/earlyx.so 16384 10 3 > gpurun_out/ab6.txt 2>&1
BRIEF=1 python tools/trace_sync.py 16384 cfd > gpurun_out/occ_ex.txt 2>&1; BRIEF=1 python tools/trace_sync.py 16384 mfd >> gpurun_out/occ_ex.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not ladder" > gpurun_out/t13.txt 2>&1; tail -2 gpurun_out/t13.txt
