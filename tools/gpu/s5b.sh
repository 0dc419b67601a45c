# session 5: half-row scan A/B on cfg4, least band height A/B on the small configs, warp-map search
mkdir -p gpurun_out
timeout 600 python tools/time_libs.py cfg4 tools/var/libbf_hs0.so paper_1803_00004_b200/libbf.so > gpurun_out/s5b_hs.txt 2>&1
cat gpurun_out/s5b_hs.txt
timeout 600 python tools/time_libs.py cfg0,cfg1,cfg3 paper_1803_00004_b200/libbf.so tools/var/libbf_th8.so tools/var/libbf_th4.so > gpurun_out/s5b_th.txt 2>&1
cat gpurun_out/s5b_th.txt
timeout 1500 python tools/wmap_search.py cfg2,cfg3,cfg1,cfg0,cfg4 1500 > gpurun_out/s5b_wmap.txt 2>&1
tail -5 gpurun_out/s5b_wmap.txt
