# one full ncu capture of synth_draws_kernel (device weight synthesis) at n = NCU_N
mkdir -p gpurun_out
N=${NCU_N:-200000000}
timeout 300 python tools/synth_time.py $N --no-check > gpurun_out/synth_pre.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:synth_draws_kernel --launch-skip 1 -c 1 \
    -o gpurun_out/synth_full -f python tools/synth_time.py $N --no-check > gpurun_out/ncu_synth.log 2>&1
