CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"warp_restrict|warp_prolongate" -o gpurun_out/prof_xfer -f $CMD > gpurun_out/ncu_xfer.log 2>&1
echo xfer=$?
