rm -f gpurun_out/x37.txt
timeout 400 python tools/time_libs.py cfg4,cfg2 tools/var/libbf_prev.so paper_1803_00004_b200/libbf.so >> gpurun_out/x37.txt 2>&1
