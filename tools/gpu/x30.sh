rm -f gpurun_out/x30.txt
for l in tm8s200 tm8; do echo "== $l" >> gpurun_out/x30.txt; CUDA_LAUNCH_BLOCKING=1 timeout 100 python tools/time_libs.py cfg0 tools/var/libbf_$l.so >> gpurun_out/x30.txt 2>&1; done
