CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:warp_restrict -c 1 -o gpurun_out/prof_restrict -f $CMD > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:warp_prolongate -s 9 -c 1 -o gpurun_out/prof_prolong -f $CMD > gpurun_out/ncu_full2.log 2>&1
echo full=$?
