for l in tm0 tms64 tmfh48; do echo "== $l" >> gpurun_out/x22.txt; CUDA_LAUNCH_BLOCKING=1 timeout 200 python tools/time_libs.py cfg0,cfg2 tools/var/libbf_$l.so >> gpurun_out/x22.txt 2>&1; done
