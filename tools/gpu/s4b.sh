# persistent partition check: cluster capacity, A/B timing against the previous build (bitwise diff), GPU tests
mkdir -p gpurun_out
./tools/microbench/clusters > gpurun_out/s4b_clusters.txt 2>&1
timeout 600 python tools/time_libs.py cfg4,cfg2,cfg1,cfg3,cfg0 tools/var/libbf_prev.so paper_1803_00004_b200/libbf.so > gpurun_out/s4b_time.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/s4b_tests.txt 2>&1
echo "tests rc $?" >> gpurun_out/s4b_tests.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k cfg4 -s > gpurun_out/s4b_full4.txt 2>&1
echo "full rc $?" >> gpurun_out/s4b_full4.txt
