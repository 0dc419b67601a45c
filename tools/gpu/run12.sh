timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed|max-abs" | head -20
for c in cfg2 cfg0 cfg1 cfg3 cfg4; do timeout 300 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline 2>&1 | tail -1 | cut -c170-230 | sed "s/^/$c /"; done
