# usage: bash tools/gpu/profile_round.sh TAG [config]
# 1) the bench line (no profiler), 2) the ncu launch list of the same command (cold-cache,
# serialised per-launch times), 3) one ncu --set full capture of the dominant kernel.
TAG=$1; CFG=${2:-cfg2}
mkdir -p gpurun_out
python -c "from paper_1803_00004_b200 import build; build.build()"
timeout 600 python bench.py --steps 10 --warmup 3 --config $CFG > gpurun_out/${TAG}_${CFG}_bench.json 2> gpurun_out/${TAG}_${CFG}_bench.err
echo "bench rc $?"; tail -c 600 gpurun_out/${TAG}_${CFG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_${CFG}_launches.csv python bench.py --steps 2 --warmup 1 --config $CFG --no-cpu-baseline \
  > gpurun_out/${TAG}_${CFG}_launches.log 2>&1
echo "launch list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bf_ -s 2 -c 1 \
  -o gpurun_out/${TAG}_${CFG} -f python bench.py --steps 1 --warmup 2 --no-cpu-baseline --config $CFG > gpurun_out/${TAG}_${CFG}_ncu.log 2>&1
echo "ncu full rc $?"
