timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/diag_fp64_pair.py c5 2>&1 | tail -3
timeout 300 python tools/diag_fp64_pair.py c3 2>&1 | tail -3
timeout 300 python tools/devtime.py c5 512 fp32 2 | tail -1
