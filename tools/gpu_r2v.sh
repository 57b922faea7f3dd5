set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in c4; do timeout 900 python tools/bulk_parity.py $c 64 2>&1 | tail -1; timeout 900 python tools/bulk_parity.py $c 64 1 2>&1 | tail -1; done
timeout 300 python tools/devtime.py c4 4096 fp32 2 nofix 2>&1 | tail -1
timeout 300 python tools/devtime.py c4 4096 fp32 2 2>&1 | tail -1
