# session 5: S-role register budget / scan unroll A/B; cfg4 map search on the current build
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2,cfg3,cfg1 paper_1803_00004_b200/libbf.so tools/var/libbf_sreg64.so tools/var/libbf_sreg80.so tools/var/libbf_su4.so tools/var/libbf_su16.so > gpurun_out/s5e_time.txt 2>&1
cat gpurun_out/s5e_time.txt
timeout 900 python tools/wmap_search.py cfg4 1500 > gpurun_out/s5e_wmap.txt 2>&1
grep -v "^ALL" gpurun_out/s5e_wmap.txt | cut -c1-200 | head -60
