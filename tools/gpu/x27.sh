rm -f gpurun_out/x27.txt
timeout 600 python tools/time_libs.py cfg2,cfg1,cfg3,cfg0 tools/var/libbf_notm.so paper_1803_00004_b200/libbf.so tools/var/libbf_fh96.so tools/var/libbf_fh104v64.so >> gpurun_out/x27.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 600 >> gpurun_out/x27.txt 2>&1
