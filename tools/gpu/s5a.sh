# session 5: warp-role map A/B (identity / balanced / balanced with an FH warp per sub-partition), then the GPU tests with durations
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg2,cfg4,cfg1,cfg3,cfg0 tools/var/libbf_wmap0.so paper_1803_00004_b200/libbf.so tools/var/libbf_wmap2.so tools/var/libbf_prev.so > gpurun_out/s5a_time.txt 2>&1
cat gpurun_out/s5a_time.txt
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 600 --durations=8 > gpurun_out/s5a_tests.txt 2>&1
echo "tests rc $?" >> gpurun_out/s5a_tests.txt
tail -15 gpurun_out/s5a_tests.txt
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -x -s --durations=8 > gpurun_out/s5a_full.txt 2>&1
echo "full rc $?" >> gpurun_out/s5a_full.txt
tail -15 gpurun_out/s5a_full.txt
