mkdir -p gpurun_out
python tools/repair_counts.py cfg4,cfg2,cfg1,cfg0 > gpurun_out/x8.txt 2>&1; python tools/repair_counts.py cfg3 12 >> gpurun_out/x8.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/x8_gputests.txt 2>&1
