rm -f gpurun_out/x28.txt
timeout 120 python tools/time_libs.py cfg2,cfg1,cfg3,cfg0 paper_1803_00004_b200/libbf.so >> gpurun_out/x28.txt 2>&1
echo "time rc=$?" >> gpurun_out/x28.txt
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 300 >> gpurun_out/x28.txt 2>&1
