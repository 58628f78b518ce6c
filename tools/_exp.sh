python -m pytest tests/test_gpu_parity.py -q -x -k "fmm or rot" 2>&1 | tail -1
for v in 1 4 8 1; do
  echo "== ml $v"; FMMBEM_ML_WARPS=$v python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phases_ms'].items()})"
done
FMMBEM_ML_WARPS=8 python -m pytest tests/test_gpu_parity.py -q -x -k "fmm or rot" 2>&1 | tail -1
