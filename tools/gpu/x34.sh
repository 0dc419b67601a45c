rm -f gpurun_out/x34.txt
timeout 400 python tools/time_libs.py cfg4,cfg2,cfg1 paper_1803_00004_b200/libbf.so tools/var/libbf_v80.so tools/var/libbf_v64.so >> gpurun_out/x34.txt 2>&1
