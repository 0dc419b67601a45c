mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/r2c_gputests.txt 2>&1
echo "rc=$?" >> gpurun_out/r2c_gputests.txt
timeout 600 python tools/gpu/diag_repair.py > gpurun_out/r2c_diag.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
BF_PARITY_OUT=gpurun_out/parity_r2c timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -rf > gpurun_out/r2c_fullsize.txt 2>&1
echo "rc=$?" >> gpurun_out/r2c_fullsize.txt
for c in cfg4 cfg2; do
  python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-per-config --config $c > gpurun_out/r2c_plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bf_ws2 -s 2 -c 1 \
    -o gpurun_out/r2c_$c -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-per-config --config $c > gpurun_out/r2c_ncu_$c.log 2>&1
done
