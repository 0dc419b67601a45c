timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "assert |FAILED|passed|failed|max-abs" | head -5
for v in 1 0; do for c in cfg2 cfg1; do BF_KERNEL=band BF_VSPLIT=$v timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline 2>&1 | tail -1 | cut -c170-230 | sed "s/^/vsplit=$v $c /"; done; done
