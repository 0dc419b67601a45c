# usage: bash tools/gpu/full.sh TAG: the whole GPU suite, then tools/gpu/iter.sh TAG
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
bash tools/gpu/iter.sh $1 ${2:-ws2}
