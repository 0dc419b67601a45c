mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg4 paper_1803_00004_b200/libbf.so tools/var/libbf_susp0.so tools/var/libbf_susp2k.so tools/var/libbf_susp.so > gpurun_out/x18.txt 2>&1
