mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2e_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/r2e_gputests.txt 2>&1
echo "rc=$?" >> gpurun_out/r2e_gputests.txt
timeout 900 python bench.py > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r2e_smoke.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2e_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r2e_ncu.log 2>&1
