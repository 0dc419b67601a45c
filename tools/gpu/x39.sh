rm -f gpurun_out/x39.txt
timeout 400 python tools/time_libs.py cfg2,cfg4,cfg1,cfg3,cfg0 tools/var/libbf_prev.so paper_1803_00004_b200/libbf.so >> gpurun_out/x39.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 300 >> gpurun_out/x39.txt 2>&1
