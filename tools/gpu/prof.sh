# usage: bash tools/gpu/prof.sh TAG [config]   (ncu full capture of one bf kernel launch)
TAG=$1; CFG=${2:-cfg2}
mkdir -p gpurun_out
python -c "from paper_1803_00004_b200 import build; build.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bf_ -s 2 -c 1 \
  -o gpurun_out/${TAG}_${CFG} -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --config $CFG > gpurun_out/${TAG}_${CFG}_ncu.log 2>&1
echo ncu rc $?
tail -3 gpurun_out/${TAG}_${CFG}_ncu.log
