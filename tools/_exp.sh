python -m pytest tests -m gpu -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_sc.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_sc.json')); print(d['ms_per_step'], d['phases_ms'], d['parity_sampled_rows'], d['e2e'], d['roofline'])"
