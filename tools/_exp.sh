for v in base "t6 96" "t6 48" "t6 192"; do
  set -- $v
  if [ $1 = base ]; then unset FMMBEM_LIB; unset FMMBEM_P2P_CHUNK; else export FMMBEM_LIB=$PWD/build/ab/libfmmbem_$1.so; export FMMBEM_P2P_CHUNK=$2; fi
  echo "== $v"; python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['phases_ms'].items()}, d['parity_sampled_rows'] if 'parity_sampled_rows' in d else '')"
done
