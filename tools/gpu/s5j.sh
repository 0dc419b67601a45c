# session 5: cluster exchange with three row slots instead of two: A/B on cfg4 (bitwise diff), under a timeout (a sync bug would hang)
mkdir -p gpurun_out
timeout 300 python tools/time_libs.py cfg4 paper_1803_00004_b200/libbf.so tools/var/libbf_xs3.so > gpurun_out/s5j_time.txt 2>&1
echo "rc $?" >> gpurun_out/s5j_time.txt
cat gpurun_out/s5j_time.txt
