for P in fp64 mixed; do
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --precision $P"
$CMD > gpurun_out/plain_$P.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:fam_tensor_apply -c 1 -o gpurun_out/prof_apply_$P -f $CMD > gpurun_out/ncu_full_$P.log 2>&1
echo $P full=$?
done
