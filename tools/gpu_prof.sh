# usage: bash tools/gpu_prof.sh <tag>   (profiles the row+col sweep kernels of both methods at 4096^2)
TAG=${1:-p}
python tools/prof_one.py mfd ${NPROF:-16384} 2 > gpurun_out/plain_mfd.log 2>&1 && python tools/prof_one.py cfd ${NPROF:-16384} 2 > gpurun_out/plain_cfd.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s 1 -c 3 -o gpurun_out/${TAG}_mfd python tools/prof_one.py mfd ${NPROF:-16384} 2 > gpurun_out/ncu_${TAG}_mfd.log 2>&1 ; \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s 1 -c 3 -o gpurun_out/${TAG}_cfd python tools/prof_one.py cfd ${NPROF:-16384} 2 > gpurun_out/ncu_${TAG}_cfd.log 2>&1 ; \
ls gpurun_out/*.ncu-rep; tail -2 gpurun_out/ncu_${TAG}_mfd.log
