# session 5, shipped build: bench line, cfg4 ncu capture (the start squarings changed its kernel), quick GPU tests
mkdir -p gpurun_out/final2
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err
echo "bench rc=$?" >> gpurun_out/final2/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bf_ws2 -s 1 -c 1 -o gpurun_out/final2/ncu_cfg4 -f python tools/run_lib.py paper_1803_00004_b200/libbf.so cfg4 2 > gpurun_out/final2/ncu_cfg4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --timeout 600 > gpurun_out/final2/tests.txt 2>&1
echo "tests rc $?" >> gpurun_out/final2/tests.txt
tail -3 gpurun_out/final2/tests.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k cfg4 -s > gpurun_out/final2/full4.txt 2>&1
echo "full rc $?" >> gpurun_out/final2/full4.txt
tail -4 gpurun_out/final2/full4.txt
head -c 600 gpurun_out/final2/bench.json
