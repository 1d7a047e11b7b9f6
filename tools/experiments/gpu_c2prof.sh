CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --config c2"
$CMD > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launches_c2.log 2>&1
echo launches=$?
