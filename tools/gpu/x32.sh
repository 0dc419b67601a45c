rm -f gpurun_out/x32.txt
timeout 200 python tools/time_libs.py cfg4,cfg2 paper_1803_00004_b200/libbf.so >> gpurun_out/x32.txt 2>&1
echo "time rc=$?" >> gpurun_out/x32.txt
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 300 >> gpurun_out/x32.txt 2>&1
