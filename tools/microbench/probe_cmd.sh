nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/microbench/fp64_probe > gpurun_out/fp64_probe.txt 2>&1
./tools/microbench/fp64_probe >> gpurun_out/fp64_probe.txt 2>&1
kill $SMI
nvidia-smi > gpurun_out/nvsmi.txt; lscpu > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt; free -g >> gpurun_out/lscpu.txt
cat gpurun_out/fp64_probe.txt
