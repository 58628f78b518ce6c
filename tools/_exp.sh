python -m pytest tests/test_gpu_parity.py -q -k "host_buffer" 2>&1 | tail -1
for v in 4 8 16 8; do
  echo "== chunks $v"; FMMBEM_E2E_CHUNKS=$v python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), d['e2e']['value'])"
done
