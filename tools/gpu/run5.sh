timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
for c in cfg0 cfg1 cfg3 cfg4; do timeout 300 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline 2>&1 | tail -1 | cut -c170-250; done
bash tools/gpu/prof.sh $1
