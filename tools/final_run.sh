#!/bin/bash
# Round-end measurement on one B200: GPU tests, smoke, the bench line, the reference arm, the ncu
# launch list of the bench command (after the same command exited 0 without ncu), a full ncu
# capture of one matvec's kernels, and the option / control workloads (analytic near field, random
# cube).  Outputs land in gpurun_out/fin_* and are summarised into profiles/.
set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_gputest.log 2>&1; tail -3 gpurun_out/fin_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; tail -c 300 gpurun_out/fin_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err; tail -c 300 gpurun_out/fin_bench_ref.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --bibee-calls 1 --no-solve > gpurun_out/fin_b_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_bench.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu --bibee-calls 1 --no-solve > gpurun_out/fin_ncu_bench.log 2>&1
timeout 300 python tools/prof_run.py --reps 2 > gpurun_out/fin_prof_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
      -k regex:"k_p2p|k_m2l_rot|k_m2m_rot|k_l2l_rot|k_p2m_t|k_l2p_t|k_m2m_sum" -s 22 -c 22 \
      -o /tmp/prof_final python tools/prof_run.py --reps 2 > gpurun_out/fin_ncu_full.log 2>&1
tail -2 gpurun_out/fin_ncu_full.log
python tools/ncu_summary.py /tmp/prof_final.ncu-rep gpurun_out/fin_ncu_full_summary.csv
ncu -i /tmp/prof_final.ncu-rep --page raw --csv > gpurun_out/fin_ncu_full_raw.csv 2>/dev/null
for k in k_p2p k_m2l_rot; do
  ncu -i /tmp/prof_final.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/fin_ncu_src_$k.csv 2>/dev/null
done
timeout 900 echo near-mode measured in tools/final_run_4gpu.sh history
timeout 900 python bench.py --config cube --steps 10 --warmup 3 > gpurun_out/fin_bench_cube.json 2> gpurun_out/fin_bench_cube.err; tail -c 200 gpurun_out/fin_bench_cube.json
ls -la gpurun_out/ | grep fin_
