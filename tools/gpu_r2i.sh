set -x
timeout 300 python tools/diag_fp64_pair.py c4
timeout 300 python tools/diag_fp64_pair.py c3
timeout 300 python tools/devtime.py c4 512 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c3 1024 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c5 256 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c3 256 fp64 2 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -12
