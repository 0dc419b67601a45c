mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/r2d_gputests.txt 2>&1
echo "rc=$?" >> gpurun_out/r2d_gputests.txt
timeout 600 python tools/gpu/diag_repair.py cfg4 cfg2 cfg1 > gpurun_out/r2d_diag.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
BF_PARITY_OUT=gpurun_out/parity_r2d timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -rf -k "cfg4 or cfg1" > gpurun_out/r2d_fullsize.txt 2>&1
echo "rc=$?" >> gpurun_out/r2d_fullsize.txt
for c in cfg4; do
  python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-per-config --config $c > gpurun_out/r2d_plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bf_ws2 -s 2 -c 1 \
    -o gpurun_out/r2d_$c -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-per-config --config $c > gpurun_out/r2d_ncu_$c.log 2>&1
done
