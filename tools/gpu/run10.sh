for n in 2 3 4; do BF_NSEG=$n timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c170-230 | sed "s/^/nseg $n /"; done
