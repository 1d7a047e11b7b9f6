# launch list of one fp64 V-cycle on c3 (ncu gpu__time_duration only) -> gpurun_out/launches_$1.csv
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain_$1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_$1.csv $CMD > gpurun_out/ncu_launches_$1.log 2>&1
echo launches_$1=$?
