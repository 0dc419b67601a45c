# session 5: bf_apply_host row chunks 4..8 (the initial state got cheaper): e2e A/B on cfg2
mkdir -p gpurun_out
timeout 900 python tools/time_host.py cfg2 paper_1803_00004_b200/libbf.so tools/var/libbf_hc4.so tools/var/libbf_hc6.so tools/var/libbf_hc7.so tools/var/libbf_hc8.so paper_1803_00004_b200/libbf.so > gpurun_out/s5k_host.txt 2>&1
cat gpurun_out/s5k_host.txt
