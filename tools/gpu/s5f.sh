# session 5 round-end evidence: GPU tests (full-size parity last), bench line, launch list, ncu captures of cfg2 / cfg4, smoke
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT
( time BF_PARITY_OUT=gpurun_out/final timeout 3000 python -m pytest tests -m gpu -q -x --timeout 2800 --durations=6 ) > gpurun_out/final/gpu_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/final/gpu_tests.txt
tail -12 gpurun_out/final/gpu_tests.txt
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
echo "bench rc=$?" >> gpurun_out/final/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/final/launches.log 2>&1
for c in cfg2 cfg4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:bf_ws2 -s 1 -c 1 -o gpurun_out/final/ncu_$c -f python tools/run_lib.py paper_1803_00004_b200/libbf.so $c 2 > gpurun_out/final/ncu_$c.log 2>&1
  ncu -i gpurun_out/final/ncu_$c.ncu-rep --page raw --csv > gpurun_out/final/ncu_${c}_raw.csv 2>&1
  ncu -i gpurun_out/final/ncu_$c.ncu-rep --page source --csv > gpurun_out/final/ncu_${c}_source.csv 2>&1
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.txt
cat gpurun_out/final/smoke.txt | tail -2
head -c 1500 gpurun_out/final/bench.json
