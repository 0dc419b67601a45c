# session 5, final tree: the whole GPU suite, smoke, bench line
mkdir -p gpurun_out/final3
cd $GRAFT_REPO_ROOT
( time timeout 3000 python -m pytest tests -m gpu -q -x --timeout 2800 --durations=5 ) > gpurun_out/final3/gpu_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/final3/gpu_tests.txt
tail -10 gpurun_out/final3/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/final3/smoke.txt
tail -2 gpurun_out/final3/smoke.txt
( time timeout 900 python bench.py ) > gpurun_out/final3/bench.json 2> gpurun_out/final3/bench.err
echo "bench rc=$?" >> gpurun_out/final3/bench.err
tail -4 gpurun_out/final3/bench.err
head -c 400 gpurun_out/final3/bench.json
