mkdir -p gpurun_out
timeout 600 python tools/time_libs.py cfg2,cfg1,cfg0,cfg3 paper_1803_00004_b200/libbf.so > gpurun_out/x20.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 600 >> gpurun_out/x20.txt 2>&1
