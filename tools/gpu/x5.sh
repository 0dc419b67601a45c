mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2 paper_1803_00004_b200/libbf.so tools/var/libbf_tlnos.so tools/var/libbf_tlnosv.so tools/var/libbf_tlnofhv.so > gpurun_out/x5_time.txt 2>&1
