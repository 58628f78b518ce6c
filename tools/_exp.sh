python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phases_ms'].items()})"
