mkdir -p gpurun_out
for v in nosfh nosv; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:bf_ws2 -s 1 -c 1 \
    -o gpurun_out/x3_$v -f python tools/run_lib.py tools/var/libbf_$v.so cfg2 2 > gpurun_out/x3_${v}_ncu.log 2>&1
  ncu -i gpurun_out/x3_$v.ncu-rep --page raw --csv > gpurun_out/x3_${v}_raw.csv 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bf_ws2 -s 1 -c 1 \
    -o gpurun_out/x3_full -f python tools/run_lib.py paper_1803_00004_b200/libbf.so cfg2 2 > gpurun_out/x3_full_ncu.log 2>&1
ncu -i gpurun_out/x3_full.ncu-rep --page raw --csv > gpurun_out/x3_full_raw.csv 2>&1
