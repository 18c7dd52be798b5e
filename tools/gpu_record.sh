# Round record on the GPU box: tests, smoke, bench (+ reference arm, shots, configs 1-3,
# the dist-local decompositions), the ncu launch list, DRAM bytes of the line kernels, L2
# bytes of config 3, one ncu --set full capture of the dominant kernel.
# Usage: TAG=r02 bash tools/gpu_record.sh
TAG=${TAG:-rec}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -2 $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --shots --steps 1000 --warmup 10 > $O/bench_shots.json 2> $O/bench_shots.err; echo "shots rc=$?"
for c in 1 2 3; do timeout 900 python bench.py --config $c > $O/bench_config$c.json 2> $O/bench_config$c.err; echo "config$c rc=$?"; done
timeout 600 python bench.py --config 1 --no-graph > $O/bench_config1_nograph.json 2>/dev/null
for m in halo transpose; do
  timeout 900 python bench.py --dist-local 4 --dist-mode $m --steps 5 --warmup 3 --no-cpu > $O/bench_distlocal4_$m.json 2> $O/bench_distlocal4_$m.err; echo "distlocal $m rc=$?"
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
for m in mfd cfd; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:adi_line_kernel --log-file $O/dram_$m.csv python tools/prof_one.py $m 16384 2 > $O/ncu_dram_$m.log 2>&1; echo "dram $m rc=$?"
done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:adi_line_kernel --log-file $O/dram_shots.csv python tools/prof_one.py shots 4096 2 > $O/ncu_dram_shots.log 2>&1; echo "dram shots rc=$?"
for m in mfd cfd; do
  timeout 600 ncu --metrics lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:adi_line_kernel --log-file $O/l2_config3_$m.csv python tools/prof_one.py $m 1601 2 > $O/ncu_l2_$m.log 2>&1; echo "l2 $m rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s 2 -c 1 \
    -o $O/full_cfd_row python tools/prof_one.py cfd 16384 2 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/full_cfd_row.ncu-rep --page raw --csv > $O/full_cfd_row_raw.csv 2>/dev/null
ls $O
