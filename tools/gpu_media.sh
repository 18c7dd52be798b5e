# Measurement of NEXT row f3 (heterogeneous media): bench --media, the ncu launch
# list, dram bytes of the media row kernels, one ncu --set full capture of the
# dominant media kernel.  Usage: TAG=r01e_media bash tools/gpu_media.sh
TAG=${TAG:-media}
set -o pipefail
mkdir -p gpurun_out/$TAG
O=gpurun_out/$TAG
timeout 900 python bench.py --media > $O/bench_media.json 2> $O/bench_media.err; echo "bench media rc=$?"
cat $O/bench_media.json; tail -2 $O/bench_media.err
timeout 900 python bench.py --media --impl reference --steps 3 > $O/bench_media_ref.json 2> $O/bench_media_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --media --steps 2 --warmup 3 --no-e2e --no-cpu > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_media.csv python bench.py --media --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
for m in mfd cfd; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:adi_line_kernel --log-file $O/dram_media_$m.csv python tools/prof_one.py $m 16384 2 media > $O/ncu_dram_$m.log 2>&1; echo "dram $m rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s 1 -c 1 \
    -o $O/full_media_cfd_row python tools/prof_one.py cfd 16384 2 media > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/full_media_cfd_row.ncu-rep --page raw --csv > $O/full_media_cfd_row_raw.csv 2>/dev/null
ls -la $O
