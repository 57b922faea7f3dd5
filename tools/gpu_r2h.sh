set -x
timeout 300 python tools/diag_cert.py c4 512
timeout 300 python tools/devtime.py c4 512 fp32 2 nofix 2>&1 | tail -1
timeout 300 python tools/devtime.py c4 512 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c5 256 fp32 2 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -12
