set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "polynomial or random_config" 2>&1 | tail -15
timeout 300 python tools/diag_flags.py 2>&1 | tail -5
