rm -f gpurun_out/sweep.txt
L=CLGEN_LIB=$PWD/build/lib_v9.so
bash tools/sweep.sh "--config c4 --num-vertices 200000000 --steps 3 --warmup 3" "$L" "$L CLGEN_CTR_HEAVY=64" "$L CLGEN_CTR_HEAVY=96" "$L CLGEN_CTR_HEAVY=192" "$L CLGEN_CTR_SPLIT=2048" "$L CLGEN_CTR_SPLIT=8192" "$L CLGEN_CTR_EPS=0.03125" "$L CLGEN_CTR_EPS=0.0078125"
