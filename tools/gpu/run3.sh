./tools/microbench/pipes4
