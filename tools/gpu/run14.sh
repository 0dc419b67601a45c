timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "assert |FAILED|passed|failed|max-abs" | head -5
for w in 0 1; do for k in band ws; do for c in cfg2 cfg1 cfg0; do BF_SCALAR_WALK=$w BF_KERNEL=$k timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline 2>&1 | tail -1 | cut -c170-230 | sed "s/^/scalar=$w $k $c /"; done; done; done
