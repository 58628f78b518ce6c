python -m pytest tests/test_gpu_parity.py -q -x -k "fmm or rot" 2>&1 | tail -2
for v in base new base new; do
  if [ $v = base ]; then export FMMBEM_LIB=$PWD/build/ab/libfmmbem_base.so; else unset FMMBEM_LIB; fi
  echo "== $v"; python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phases_ms'].items()})"
done
