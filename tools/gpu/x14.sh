mkdir -p gpurun_out
timeout 900 python tools/time_cached.py paper_1803_00004_b200/libbf.so > gpurun_out/x14.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "case1 or cache" --timeout 600 >> gpurun_out/x14.txt 2>&1
