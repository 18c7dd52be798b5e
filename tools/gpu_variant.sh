# Measurement of a NEXT-row variant: bench line, reference arm, ncu launch list, dram
# bytes of its line kernels, one ncu --set full capture of its row kernel.
# Usage: TAG=r01e_full FLAG=--full M=cfd_full PM=media|"" bash tools/gpu_variant.sh
TAG=${TAG:-variant}; FLAG=${FLAG:---full}; M=${M:-cfd_full}; PM=${PM:-}
set -o pipefail
mkdir -p gpurun_out/$TAG
O=gpurun_out/$TAG
timeout 900 python bench.py $FLAG > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json; tail -2 $O/bench.err
timeout 900 python bench.py $FLAG --impl reference --steps 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py $FLAG --steps 2 --warmup 3 --no-e2e --no-cpu > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py $FLAG --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:adi_line_kernel --log-file $O/dram_$M.csv python tools/prof_one.py $M 16384 2 $PM > $O/ncu_dram.log 2>&1; echo "dram rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adi_line_kernel -s 2 -c 1 \
    -o $O/full_${M}_row python tools/prof_one.py $M 16384 2 $PM > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/full_${M}_row.ncu-rep --page raw --csv > $O/full_${M}_row_raw.csv 2>/dev/null
ls -la $O
