mkdir -p gpurun_out
timeout 900 python tools/time_cached.py tools/var/libbf_c992nc.so tools/var/libbf_c992k1.so > gpurun_out/x13.txt 2>&1
