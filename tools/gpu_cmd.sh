NCU_SKIP=0 bash tools/ncu_capture.sh v12walk ctr_walk_kernel --config c4 --num-vertices 200000000 --steps 1 --warmup 0
