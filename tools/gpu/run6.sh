timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for n in 2 4; do BF_NSEG=$n timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c170-230; done
for c in cfg0 cfg1 cfg3 cfg4; do timeout 300 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline 2>&1 | tail -1 | cut -c170-230; done
bash tools/gpu/prof.sh $1
