timeout 300 python tools/diag_flags.py c4 512 2>&1 | head -4
timeout 300 python tools/diag_flags.py c5 64 2>&1 | head -4
