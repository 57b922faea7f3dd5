set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/devtime.py c4 4096 fp32 2 2>&1 | tail -1
timeout 900 python tools/bulk_parity.py c4 64 5 2>&1 | tail -1
timeout 900 python tools/bulk_parity.py c4 64 6 2>&1 | tail -1
