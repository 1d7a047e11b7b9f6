# launch lists (one V-cycle, both precisions) + ncu --set full of the fp32 apply
for P in fp64 mixed; do
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --precision $P"
$CMD > gpurun_out/plain_$P.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_$P.csv $CMD > gpurun_out/ncu_launches_$P.log 2>&1
echo launches_$P=$?
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --precision mixed"
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:fam_tensor_apply -c 1 -o gpurun_out/prof_apply_f32 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo full=$?
