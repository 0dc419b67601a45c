mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2 paper_1803_00004_b200/libbf.so tools/var/libbf_now.so tools/var/libbf_nolds.so tools/var/libbf_fh.so tools/var/libbf_fhnow.so tools/var/libbf_fhnolds.so > gpurun_out/x6_time.txt 2>&1
