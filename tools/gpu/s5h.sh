# session 5: cost-model weight of the (now cooperative) initial state: A/B over the five configs
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg4,cfg2,cfg1,cfg3,cfg0 paper_1803_00004_b200/libbf.so tools/var/libbf_is5.so tools/var/libbf_is3.so > gpurun_out/s5h_time.txt 2>&1
cat gpurun_out/s5h_time.txt
