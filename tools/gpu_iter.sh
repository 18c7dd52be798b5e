# one iteration on the GPU box: parity tests, quick bench, tile trace
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -6
timeout 600 python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json'))
print('value %.3e'%d['value'], 'ms/step %.2f'%d['ms_per_step'])
for m,v in d['per_method'].items(): print(m, 'ms/step %.2f'%v['ms_per_step'], 'hbm_frac %.3f'%v['hbm_frac_step'], {k: round(x,3) for k,x in v['kernel_avg_ms'].items()})
print(d['roofline']); print(d['clocks'])
" 2>&1 | tail -8
tail -3 gpurun_out/bench_quick.err
[ -n "$TRACE" ] && timeout 600 python tools/tile_trace.py 16384 gpurun_out/trace/t 2>&1 | grep "persist=0" ; rm -rf gpurun_out/trace
