rm -f gpurun_out/x29.txt
timeout 300 python tools/time_libs.py cfg2,cfg1,cfg3 paper_1803_00004_b200/libbf.so tools/var/libbf_v80.so >> gpurun_out/x29.txt 2>&1
