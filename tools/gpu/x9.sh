mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg4 paper_1803_00004_b200/libbf.so tools/var/libbf_c4nov.so tools/var/libbf_c4nofh.so tools/var/libbf_c4nos.so tools/var/libbf_c4now.so > gpurun_out/x9_time.txt 2>&1
timeout 1200 python tools/bench_extras.py --json gpurun_out/x9_extras.json > gpurun_out/x9_extras.txt 2>&1
