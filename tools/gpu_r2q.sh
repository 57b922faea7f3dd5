timeout 600 python tools/diag_cert.py c4 1024
cd ab/r1 && for c in "c5 512" "c3 1024"; do timeout 300 python tools/devtime.py $c fp32 2 2>&1 | tail -1; done; cd ../..
for c in "c5 512" "c3 1024"; do timeout 300 python tools/devtime.py $c fp32 2 nofix 2>&1 | tail -1; done
