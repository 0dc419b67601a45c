for w in "cfg3" "cfg0_f32" "cfg0 16" "cfg1 8" "cfg0"; do CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/tmtest.py $w >> gpurun_out/x21.txt 2>&1; done
