# ncu --set full of the row sweep kernel of one method (default mfd) at 16384^2
M=${1:-mfd}; TAG=${2:-p}
python tools/prof_one.py $M ${NPROF:-16384} 2 > gpurun_out/plain_$M.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s ${SKIP:-2} -c 1 -o gpurun_out/${TAG}_$M python tools/prof_one.py $M ${NPROF:-16384} 2 > gpurun_out/ncu_${TAG}_$M.log 2>&1
tail -2 gpurun_out/ncu_${TAG}_$M.log
