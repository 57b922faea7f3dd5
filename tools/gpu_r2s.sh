for r in 1 2; do
SK_LIB_OVERRIDE=ab/vC.so timeout 300 python tools/devtime.py c5 512 fp32 2 nofix 2>&1 | tail -1
timeout 300 python tools/devtime.py c5 512 fp32 2 nofix 2>&1 | tail -1
done
