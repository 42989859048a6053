# A/B lines only (no tests): each arg is an env assignment list
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
bash tools/ab_blk.sh "${@}"
cat gpurun_out/ab.log
