mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_fullsize.py --timeout 600 -x > gpurun_out/r2b_gputests.txt 2>&1
echo "rc=$?" >> gpurun_out/r2b_gputests.txt
timeout 600 python tools/gpu/diag_repair.py > gpurun_out/r2b_diag.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
