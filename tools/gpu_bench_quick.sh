timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bq.json 2> gpurun_out/bq.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bq.json'))
print('value %.3e'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], 'cpu', d['cpu_baseline'])
for m,v in d['per_method'].items(): print(m, 'ms/step %.2f'%v['ms_per_step'], 'hbm_frac %.3f'%v['hbm_frac_step'])
print(d['roofline'])"
tail -3 gpurun_out/bq.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bq_tr.json 2> gpurun_out/bq_tr.err; echo "torchrun rc=$?"; head -c 300 gpurun_out/bq_tr.json; tail -2 gpurun_out/bq_tr.err
