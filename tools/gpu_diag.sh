# Diagnosis of the line kernels on the GPU box: sweep-cost fit, tile timeline, and one
# ncu --set full capture of each method's interior row launch.  TAG=x bash tools/gpu_diag.sh
TAG=${TAG:-diag}; O=gpurun_out/$TAG; mkdir -p $O
timeout 300 python tools/sweep_cost.py 16384 > $O/sweep_cost.txt 2>&1; cat $O/sweep_cost.txt
timeout 300 python tools/tile_trace.py 16384 $O/trace/t > $O/tile_trace.txt 2>&1; cat $O/tile_trace.txt; rm -rf $O/trace
for M in cfd mfd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s 2 -c 1 \
      -o $O/full_${M}_row python tools/prof_one.py $M 16384 2 > $O/ncu_$M.log 2>&1; echo "ncu $M rc=$?"
done
