# ncu --set full of the fused chunk kernel (finest level, first two launches of one V-cycle)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:chunk_apply -c 2 -o gpurun_out/prof_chunk -f $CMD > gpurun_out/ncu_full.log 2>&1
echo full=$?
