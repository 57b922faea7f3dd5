timeout 300 python tools/devtime.py L256d4M8 4096 fp32 2 0 nofix | tail -1
timeout 300 python tools/devtime.py L512d4M8 2048 fp32 2 0 nofix | tail -1
timeout 300 python tools/devtime.py c5 512 fp32 2 0 nofix | tail -1
timeout 300 python tools/devtime.py c5 512 fp32 2 | tail -1
