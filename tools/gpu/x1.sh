mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2,cfg1 paper_1803_00004_b200/libbf.so tools/var/libbf_nov.so tools/var/libbf_nos.so tools/var/libbf_nofh.so tools/var/libbf_nofhv.so > gpurun_out/x1_time.txt 2>&1
timeout 600 python bench.py --no-per-config --no-cpu-baseline > gpurun_out/x1_bench.json 2> gpurun_out/x1_bench.err
