# GPU check used during development: parity tests + quick device timings
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for a in "$@"; do timeout 300 python tools/devtime.py $a 2>&1 | tail -2; done
