mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bf_cached -s 1 -c 1 -o gpurun_out/x15_cached -f python tools/time_cached.py paper_1803_00004_b200/libbf.so > gpurun_out/x15.log 2>&1
ncu -i gpurun_out/x15_cached.ncu-rep --page raw --csv > gpurun_out/x15_raw.csv 2>&1
