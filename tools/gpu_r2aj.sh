timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k certification_flags 2>&1 | grep -E "^E|assert|Error" | head -20
timeout 900 python tools/bulk_parity.py c4 64 6 2>&1 | tail -1
