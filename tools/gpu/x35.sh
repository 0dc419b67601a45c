rm -f gpurun_out/x35.txt
timeout 400 python tools/time_libs.py cfg2,cfg1,cfg3,cfg0,cfg4 paper_1803_00004_b200/libbf.so tools/var/libbf_v56.so tools/var/libbf_v88.so >> gpurun_out/x35.txt 2>&1
