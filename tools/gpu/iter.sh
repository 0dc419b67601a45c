# usage: bash tools/gpu/iter.sh TAG [KERNEL]: bitwise-agreement tests, benches of KERNEL on cfg2/1/0/3,
# one ncu --set full capture of cfg2
TAG=$1; K=${2:-ws2}
timeout 600 python -m pytest tests -m gpu -q -x -k "agree or exact" 2>&1 | tail -2
for c in cfg2 cfg1 cfg0 cfg3; do BF_KERNEL=$K timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*' | sed "s/^/$K $c /"; done
bash tools/gpu/ncu_one.sh $TAG cfg2 $K
