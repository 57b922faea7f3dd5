set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python tools/devtime.py c4 2048 fp32 1 > gpurun_out/r2_c4_launches.log 2>&1
python tools/ncu_launches.py gpurun_out/r2_c4_launches.csv > gpurun_out/r2_c4_launches.txt 2>&1; cat gpurun_out/r2_c4_launches.txt | head -30
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c3_launches.csv python tools/devtime.py c3 2048 fp32 1 > gpurun_out/r2_c3_launches.log 2>&1
python tools/ncu_launches.py gpurun_out/r2_c3_launches.csv > gpurun_out/r2_c3_launches.txt 2>&1; cat gpurun_out/r2_c3_launches.txt | head -30
