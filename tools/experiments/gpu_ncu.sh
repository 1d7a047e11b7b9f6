# launch list of one V-cycle + ncu --set full of the finest-level operator apply (1 GPU)
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:fam_tensor_apply -c 2 -o gpurun_out/prof_apply -f $CMD > gpurun_out/ncu_full.log 2>&1
echo full=$?
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:cheb_step -c 1 -o gpurun_out/prof_cheb -f $CMD > gpurun_out/ncu_full2.log 2>&1
echo full2=$?
