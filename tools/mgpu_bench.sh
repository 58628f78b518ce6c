for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --no-cpu 2>gpurun_out/err$N.txt | tail -1 > gpurun_out/bench_n$N.json; python -c "import json; d=json.load(open('gpurun_out/bench_n$N.json')); print('N$N', round(d['ms_per_step'],2), d['value'], d['e2e']['value'], d.get('comm_ms'), d['clocks'])"
done
