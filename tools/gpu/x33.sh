rm -f gpurun_out/x33.txt
timeout 300 python tools/time_libs.py cfg4 paper_1803_00004_b200/libbf.so tools/var/libbf_pf72.so >> gpurun_out/x33.txt 2>&1
