timeout 900 python -m pytest tests -m gpu -q -x -k "agree or exact or rank2 or narrow or small or multi or degenerate" 2>&1 | tail -2
for k in band ws ws2; do for c in cfg2 cfg1 cfg0 cfg3; do BF_KERNEL=$k timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline 2>&1 | tail -1 | cut -c170-230 | sed "s/^/$k $c /"; done; done
