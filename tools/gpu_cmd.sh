rm -f gpurun_out/sweep.txt
bash tools/sweep.sh "--config c4 --steps 2 --warmup 3" "CLGEN_CTR_HEAVY=256" "CLGEN_CTR_HEAVY=384" "CLGEN_CTR_HEAVY=512" "CLGEN_CTR_HEAVY=256 CLGEN_CTR_SPLIT=8192" "CLGEN_CTR_HEAVY=384 CLGEN_CTR_SPLIT=8192"
bash tools/sweep.sh "--config c3 --steps 5 --warmup 3" "X=1" "CLGEN_CTR_HEAVY=256" "CLGEN_CTR_HEAVY=384"
bash tools/sweep.sh "--config c5 --steps 5 --warmup 3" "X=1" "CLGEN_CTR_HEAVY=256" "CLGEN_CTR_HEAVY=384"
