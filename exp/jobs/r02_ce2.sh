export BURST_BENCH_ONE_GPU=1 BURST_BENCH_BACKEND=gloo
for cfg in c2 c3; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --config $cfg --comm ce --skip-cpu > gpurun_out/r02_bench_ce2_$cfg.json 2> gpurun_out/r02_bench_ce2_$cfg.err
done
for cfg in c2 c3; do python -c "
import json,sys; d=json.loads([l for l in open('gpurun_out/r02_bench_ce2_$cfg.json') if l.startswith('{')][0]); print('$cfg', d['value'], d['ms_per_step'], json.dumps(d['comm']))"; done
