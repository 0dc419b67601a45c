# session 5: V role register budget under the new warp-role map (56 / 64 / 72)
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2,cfg3,cfg1 paper_1803_00004_b200/libbf.so tools/var/libbf_v56.so tools/var/libbf_v72.so > gpurun_out/s5n_time.txt 2>&1
grep -v diff gpurun_out/s5n_time.txt
