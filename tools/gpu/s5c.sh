# session 5: new default map vs identity (all configs), half-row scan A/B under the new map, search again (all results kept)
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2,cfg4,cfg1,cfg3,cfg0 tools/var/libbf_prev.so paper_1803_00004_b200/libbf.so tools/var/libbf_wmap0.so tools/var/libbf_hs0.so > gpurun_out/s5c_time.txt 2>&1
cat gpurun_out/s5c_time.txt
timeout 1500 python tools/wmap_search.py cfg1,cfg4,cfg2,cfg3,cfg0 1500 > gpurun_out/s5c_wmap.txt 2>&1
grep -v "^  \|^ALL" gpurun_out/s5c_wmap.txt | cut -c1-300
