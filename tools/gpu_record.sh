# Round record: tests, bench (+reference arm), ncu launch list, dram bytes of the
# row kernels, one ncu --set full capture of the dominant kernel.  Usage: TAG=r01b bash tools/gpu_record.sh
TAG=${TAG:-rec}
set -o pipefail
mkdir -p gpurun_out/$TAG
O=gpurun_out/$TAG
timeout 900 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json; tail -2 $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
cat $O/bench_ref.json
timeout 900 python bench.py --shots --steps 1000 --warmup 10 > $O/bench_shots.json 2> $O/bench_shots.err; echo "shots rc=$?"
cat $O/bench_shots.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
for m in mfd cfd; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:adi_line_kernel --log-file $O/dram_$m.csv python tools/prof_one.py $m 16384 2 > $O/ncu_dram_$m.log 2>&1; echo "dram $m rc=$?"
done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:adi_line_kernel --log-file $O/dram_shots.csv python tools/prof_one.py shots 4096 2 > $O/ncu_dram_shots.log 2>&1; echo "dram shots rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s 2 -c 1 \
    -o $O/full_cfd_row python tools/prof_one.py cfd 16384 2 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/full_cfd_row.ncu-rep --page raw --csv > $O/full_cfd_row_raw.csv 2>/dev/null
ls -la $O
