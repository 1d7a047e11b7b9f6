CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:fam_tensor_apply -c 1 -o gpurun_out/prof_apply2 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo full=$?
