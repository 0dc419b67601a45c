rm -f gpurun_out/x38.txt
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 300 >> gpurun_out/x38.txt 2>&1
