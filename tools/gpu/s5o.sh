# session 5: where the idle warps sit inside a sub-partition (last / first / third slot), on the best layouts
mkdir -p gpurun_out
timeout 1200 python tools/wmap_search.py cfg1,cfg2,cfg3 1500 > gpurun_out/s5o_wmap.txt 2>&1
grep -v "^ALL" gpurun_out/s5o_wmap.txt | grep -A14 "second pass\|default" | cut -c1-150
