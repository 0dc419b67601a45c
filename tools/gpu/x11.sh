mkdir -p gpurun_out
timeout 900 python tools/time_cached.py paper_1803_00004_b200/libbf.so tools/var/libbf_c256k4.so tools/var/libbf_c512k4.so tools/var/libbf_c768k2.so > gpurun_out/x11.txt 2>&1
