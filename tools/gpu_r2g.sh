set -x
timeout 300 python tools/diag_fp64_pair.py c4
timeout 300 python tools/diag_fp64_pair.py c5
timeout 300 python tools/diag_fp64_pair.py c3
timeout 300 python tools/diag_cert.py c4 512
