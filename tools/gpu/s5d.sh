# session 5: cooperative initial state (all warps) vs the previous build: bitwise diff, times, GPU tests; map search on the new build
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2,cfg4,cfg1,cfg3,cfg0 tools/var/libbf_prev.so paper_1803_00004_b200/libbf.so > gpurun_out/s5d_time.txt 2>&1
cat gpurun_out/s5d_time.txt
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/s5d_tests.txt 2>&1
echo "tests rc $?" >> gpurun_out/s5d_tests.txt
tail -5 gpurun_out/s5d_tests.txt
timeout 900 python tools/wmap_search.py cfg1,cfg2,cfg3 1500 > gpurun_out/s5d_wmap.txt 2>&1
grep -v "^  \|^ALL" gpurun_out/s5d_wmap.txt | cut -c1-300
