set -x
timeout 300 python tools/devtime.py c5 64 fp32 2 nofix 2>&1 | tail -2
timeout 300 python tools/devtime.py c5 64 fp32 2 2>&1 | tail -2
timeout 300 python tools/devtime.py c3 1024 fp32 2 nofix 2>&1 | tail -1
timeout 300 python tools/devtime.py c3 1024 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c4 512 fp32 2 nofix 2>&1 | tail -1
timeout 300 python tools/devtime.py c4 512 fp32 2 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -12
