timeout 300 python tools/diag_flags.py c5 512 2>&1 | tail -8
timeout 300 python tools/diag_flags.py c2 512 2>&1 | tail -4
