rm -f gpurun_out/x36.txt
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 300 >> gpurun_out/x36.txt 2>&1
for c in cfg2 cfg4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:bf_ws2 -s 1 -c 1 -o gpurun_out/x36_$c -f python tools/run_lib.py paper_1803_00004_b200/libbf.so $c 2 > gpurun_out/x36_ncu_$c.log 2>&1
  ncu -i gpurun_out/x36_$c.ncu-rep --page raw --csv > gpurun_out/x36_${c}_raw.csv 2>&1
done
