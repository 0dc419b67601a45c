mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "case1 or cache or graph" --timeout 600 > gpurun_out/x10_tests.txt 2>&1
timeout 600 python tools/bench_extras.py case1 > gpurun_out/x10_extras.txt 2>&1
