#!/bin/bash
# Round-end measurement on one B200: GPU tests, smoke, the bench line, the reference arm, the ncu
# launch list of the bench command (after the same command exited 0 without ncu) and a full ncu
# capture of one matvec's kernels.  Outputs land in gpurun_out/ and are summarised into profiles/.
set -x
python -m pytest tests -m gpu -q > gpurun_out/final_gputest.log 2>&1; tail -3 gpurun_out/final_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
python bench.py --steps 2 --warmup 3 --no-cpu --bibee-calls 1 > gpurun_out/b_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu --bibee-calls 1 > gpurun_out/ncu_bench.log 2>&1
python tools/prof_run.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"k_p2p|k_m2l_rot|k_m2m_rot|k_l2l_rot|k_p2m_t|k_l2p_t|k_m2m_sum" -s 22 -c 22 \
      -o /tmp/prof_final python tools/prof_run.py --reps 2 > gpurun_out/ncu_full_final.log 2>&1
tail -2 gpurun_out/ncu_full_final.log
# the report itself stays on the box (gpurun_out must stay under 64 MiB): summaries only
python tools/ncu_summary.py /tmp/prof_final.ncu-rep gpurun_out/ncu_full_final_summary.csv
ncu -i /tmp/prof_final.ncu-rep --page raw --csv > gpurun_out/ncu_full_final_raw.csv 2>/dev/null
for k in k_p2p k_m2l_rot; do
  ncu -i /tmp/prof_final.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/ncu_src_$k.csv 2>/dev/null
done
./tools/micro/ffma2_probe > gpurun_out/ffma2_probe.txt 2>&1
ls -la gpurun_out/
