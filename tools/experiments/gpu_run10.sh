timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log
for P in fp64 mixed; do
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --precision $P"
$CMD > gpurun_out/plain_$P.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_$P.csv $CMD > gpurun_out/ncu_launches_$P.log 2>&1
echo launches_$P=$?
done
