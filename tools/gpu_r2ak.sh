set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/devtime.py c4 4096 fp32 2 2>&1 | tail -1
for s in 6 7 8 9; do timeout 900 python tools/bulk_parity.py c4 64 $s 2>&1 | tail -1; done
timeout 300 python tools/diag_fp64_pair.py c4 2>&1 | tail -3
timeout 300 python tools/devtime.py c4 512 fp64 2 2>&1 | tail -1
