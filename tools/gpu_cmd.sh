timeout 900 python -m pytest tests/test_gpu_counter.py -q -x > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
bash tools/ab.sh "--config c4 --num-vertices 200000000 --steps 3 --warmup 3" build/lib_v9.so build/lib_v10.so build/lib_v10.so:CLGEN_L2_FETCH=32
