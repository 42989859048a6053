timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tall.log 2>&1; echo rc=$? >> gpurun_out/tall.log
rm -f gpurun_out/sweep.txt
bash tools/sweep.sh "--config c4 --num-vertices 200000000 --steps 3 --warmup 3" "CLGEN_LIB=$PWD/build/lib_v13.so"
bash tools/sweep.sh "--config c3 --steps 5 --warmup 3" "CLGEN_LIB=$PWD/build/lib_v13.so"
bash tools/sweep.sh "--config c5 --steps 5 --warmup 3" "CLGEN_LIB=$PWD/build/lib_v13.so"
