rm -f gpurun_out/x25.txt
for l in tmw0 tmnod tmc512; do echo "== $l" >> gpurun_out/x25.txt; CUDA_LAUNCH_BLOCKING=1 timeout 200 python tools/time_libs.py cfg0 tools/var/libbf_$l.so >> gpurun_out/x25.txt 2>&1; done
