# ncu --set full of the fused prolongation + first post-smoothing step (TA_CHEB_P01) and of TA_CHEB_01-free mode 5 for comparison
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    --kernel-name-base demangled -k "regex:fam_tensor_apply<.int.2, double, .int.6>" -s 9 -c 1 -o gpurun_out/prof_p01 -f $CMD > gpurun_out/ncu_p01.log 2>&1
echo p01=$?
ncu --set full --clock-control none --import-source on --profile-from-start off \


