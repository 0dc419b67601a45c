set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err; echo bench rc $?
cat gpurun_out/bench_v5.json
for c in cfg0 cfg1 cfg3 cfg4; do timeout 300 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bench_v5_$c.json 2>&1; tail -1 gpurun_out/bench_v5_$c.json | cut -c1-300; done
