set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/devtime.py c5 512 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c3 1024 fp32 2 2>&1 | tail -1
for c in c3 c5 c2 c4; do timeout 900 python tools/bulk_parity.py $c 64 2>&1 | tail -1; done
