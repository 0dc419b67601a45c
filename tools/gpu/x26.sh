rm -f gpurun_out/x26.txt
CUDA_LAUNCH_BLOCKING=1 timeout 200 python tools/time_libs.py cfg0,cfg2 tools/var/libbf_tmsm.so >> gpurun_out/x26.txt 2>&1
