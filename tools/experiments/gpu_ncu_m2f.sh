CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --precision mixed"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    --kernel-name-base demangled -k "regex:fam_tensor_apply<.int.2, float, .int.2>" -c 1 -o gpurun_out/prof_m2f -f $CMD > gpurun_out/ncu_m2f.log 2>&1
echo m2f=$?
