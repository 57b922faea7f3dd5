timeout 900 python -m pytest tests -m gpu -q -x -k "pde" 2>&1 | tail -3
timeout 600 python tools/measure_aux.py 2>&1 | head -12
