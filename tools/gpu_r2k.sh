set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/devtime.py c4 4096 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c3 8192 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c3 8192 fp32 2 nofix 2>&1 | tail -1
