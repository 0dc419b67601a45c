# usage: bash tools/gpu/ncu_one.sh TAG CFG [BF_KERNEL]: one ncu --set full capture of the bf_ kernel
TAG=$1; CFG=${2:-cfg2}; export BF_KERNEL=${3:-}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bf_ -s 2 -c 1 \
  -o gpurun_out/${TAG} -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --config $CFG > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc $?"
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
