python -m pytest tests/test_gpu_parity.py -q -k "host_buffer" 2>&1 | grep -E "passed|failed|assert|Error" | head
