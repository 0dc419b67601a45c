mkdir -p gpurun_out
timeout 900 python tools/time_cached.py paper_1803_00004_b200/libbf.so tools/var/libbf_k512x4.so tools/var/libbf_k256x8.so > gpurun_out/x16.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "case1 or cache" --timeout 600 >> gpurun_out/x16.txt 2>&1
