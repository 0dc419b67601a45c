# Refresh the committed measurements: cfg2 bench + launch list + full capture, the extras table,
# and the cfg4 bench line.
set -x
bash tools/gpu/profile_round.sh r1_final2 cfg2
timeout 600 python tools/bench_extras.py > gpurun_out/r1_final2_extras.txt 2>&1; echo "extras rc $?"
timeout 600 python bench.py --steps 5 --warmup 3 --config cfg4 --no-cpu-baseline > gpurun_out/r1_final2_cfg4_bench.json 2>&1; echo "cfg4 rc $?"
ncu -i gpurun_out/r1_final2_cfg2.ncu-rep --page raw --csv > gpurun_out/r1_final2_cfg2_raw.csv 2>&1
ncu -i gpurun_out/r1_final2_cfg2.ncu-rep --page source --csv --print-source sass > gpurun_out/r1_final2_cfg2_sass.csv 2>&1
ls -la gpurun_out
