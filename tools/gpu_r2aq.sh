timeout 300 python tools/devtime.py c4 4096 fp32 2 0 nofix | tail -1
timeout 300 python tools/devtime.py c4 4096 fp32 2 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python tools/devtime.py c4 1024 fp32 1 > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/r2_c4_launches.csv > gpurun_out/r2_c4_launches.txt 2>&1; head -14 gpurun_out/r2_c4_launches.txt
