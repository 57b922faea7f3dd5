set -x
timeout 300 python tools/diag_cert.py c5 8
timeout 300 python tools/diag_cert.py c4 32
timeout 300 python tools/diag_cert.py c3 16
timeout 300 python tools/diag_cert.py c2 32
timeout 900 python -m pytest tests -m gpu -q -x -k "random_config_matches_oracle and 180 or symmetric_equals_cross or full_size_baseline_configs and c2n" 2>&1 | grep -E "Error|error|assert|^E" | head -40
