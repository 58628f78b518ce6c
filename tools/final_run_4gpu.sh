#!/bin/bash
# Round-end multi-GPU measurement on one 4-GPU box: the 2-GPU parity tests, the parity check at 4
# ranks, the C5 bench at 2 and 4 GPUs and the 22^3 array (1.09e9 panels) at 4 GPUs.  Outputs land
# in gpurun_out/fin4_* and are summarised into profiles/.
set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q > gpurun_out/fin4_mgpu_tests.log 2>&1; tail -3 gpurun_out/fin4_mgpu_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 tools/mgpu_check.py c3 > gpurun_out/fin4_mgpu_c3_n4.log 2>&1; echo mgpu4 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/fin4_bench_n2.log 2>&1; echo n2 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29663 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/fin4_bench_n4.log 2>&1; echo n4 $?
FMMBEM_VERBOSE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29664 bench.py --gpus 4 --config c5_22 --steps 5 --warmup 3 > gpurun_out/fin4_bench_c5_22_n4.log 2>&1; echo c5_22 $?
