cd tools/microbench && for f in pipes pipes2 pipes3; do ./$f; done > ../../gpurun_out/pipes.txt 2>&1; cd ../..
cat gpurun_out/pipes.txt
bash tools/gpu/prof.sh v5
