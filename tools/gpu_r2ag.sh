set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/devtime.py c4 1024 fp32 3 | tail -1
timeout 300 python tools/devtime.py c4 4096 fp32 2 | tail -1
timeout 900 python tools/bulk_parity.py c4 64 4 | tail -1
