set -x
mkdir -p gpurun_out
timeout 2000 python tools/calib_fp32_error.py 500 7 > gpurun_out/calib7.jsonl 2> gpurun_out/calib7.err
wc -l gpurun_out/calib7.jsonl; tail -3 gpurun_out/calib7.err
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -8
