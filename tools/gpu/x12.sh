mkdir -p gpurun_out
timeout 900 python tools/time_cached.py tools/var/libbf_c768k2.so tools/var/libbf_c992k2.so tools/var/libbf_c768k2s10.so > gpurun_out/x12.txt 2>&1
