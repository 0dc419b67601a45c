# session 5: power-of-two start squarings as straight-line code: A/B against the profiled build (bitwise diff)
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg4,cfg2,cfg3 tools/var/libbf_s5f.so paper_1803_00004_b200/libbf.so > gpurun_out/s5g_time.txt 2>&1
cat gpurun_out/s5g_time.txt
timeout 900 python -m pytest tests/test_gpu_contract.py -m gpu -q -x --timeout 600 -k "cluster or bitwise or graph" > gpurun_out/s5g_tests.txt 2>&1
tail -3 gpurun_out/s5g_tests.txt
