CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:warp_restrict -c 1 -o gpurun_out/prof_restrict2 -f $CMD > gpurun_out/ncu_r2.log 2>&1
echo r=$?
