# session 5: TMEM batch prefetch in the V role (next batch loaded during the current one), V at 64 / 72 / 80 registers
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2,cfg4,cfg3,cfg1 paper_1803_00004_b200/libbf.so tools/var/libbf_pf.so tools/var/libbf_pf72.so tools/var/libbf_pf80.so > gpurun_out/s5l_time.txt 2>&1
cat gpurun_out/s5l_time.txt
