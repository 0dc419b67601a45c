# session-4 profiles of the shipped build: ncu --set full of kernel 2b on cfg4 and cfg2, launch list on cfg2
mkdir -p gpurun_out
bash tools/gpu/ncu_one.sh s4_cfg4 cfg4
bash tools/gpu/ncu_one.sh s4_cfg2 cfg2
ncu -i gpurun_out/s4_cfg4.ncu-rep --page source --csv > gpurun_out/s4_cfg4_source.csv 2>&1
ncu -i gpurun_out/s4_cfg2.ncu-rep --page source --csv > gpurun_out/s4_cfg2_source.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/s4_cfg2_launches.csv python bench.py --steps 2 --warmup 3 --config cfg2 --no-cpu-baseline --no-per-config \
  > gpurun_out/s4_launches.log 2>&1
echo "launch list rc $?"
