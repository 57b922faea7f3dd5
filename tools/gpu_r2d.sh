set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25
timeout 600 python tools/devtime.py c3 1024 fp32 3 2>&1 | tail -3
timeout 600 python tools/devtime.py c5 256 fp32 2 2>&1 | tail -2
timeout 600 python tools/devtime.py c2 1024 fp32 2 2>&1 | tail -2
