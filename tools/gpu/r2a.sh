mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/r2a_gputests.txt 2>&1
echo "rc=$?" >> gpurun_out/r2a_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
BF_PARITY_OUT=gpurun_out/parity timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -rf > gpurun_out/r2a_fullsize.txt 2>&1
echo "rc=$?" >> gpurun_out/r2a_fullsize.txt
