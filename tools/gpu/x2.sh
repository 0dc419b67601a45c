mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2 paper_1803_00004_b200/libbf.so tools/var/libbf_nosv.so tools/var/libbf_nosfh.so > gpurun_out/x2_time.txt 2>&1
