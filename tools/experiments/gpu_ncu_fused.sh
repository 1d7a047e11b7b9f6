# ncu --set full of the fused operator kernels on the finest level (fp64): TA_CHEB_11 (first launch) and TA_CHEB_P01 (last launch)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    --kernel-name-base demangled -k "regex:fam_tensor_apply<.int.2, double, .int.2>" -c 1 -o gpurun_out/prof_fused11 -f $CMD > gpurun_out/ncu_f11.log 2>&1
echo f11=$?
ncu --set full --clock-control none --import-source on --profile-from-start off \
    --kernel-name-base demangled -k "regex:fam_tensor_apply<.int.2, double, .int.6>" -s 9 -c 1 -o gpurun_out/prof_fusedp01 -f $CMD > gpurun_out/ncu_fp01.log 2>&1
echo fp01=$?
