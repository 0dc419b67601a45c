rm -f gpurun_out/x23.txt
for l in tminit0 tmrow0 tmboth0; do echo "== $l" >> gpurun_out/x23.txt; CUDA_LAUNCH_BLOCKING=1 timeout 200 python tools/time_libs.py cfg0 tools/var/libbf_$l.so >> gpurun_out/x23.txt 2>&1; done
