timeout 900 python -m pytest tests -m gpu -q -x -k "rfsf or lifted or feature" 2>&1 | tail -3
timeout 600 python tools/measure_aux.py 2>&1 | sed -n '/rfsf_exact_gram/,+6p'
