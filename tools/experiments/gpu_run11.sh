timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log
for W in 512 1024 2048; do
GMG_LAG_W=$W timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_w$W.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_w$W.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('W=$W', d['dtype'], d['ms_per_step'], '%.3g'%d['value'])"
done
timeout 600 python bench.py --no-cpu-baseline --steps 30 --precision mixed > gpurun_out/bench_mixed.log 2>&1
tail -1 gpurun_out/bench_mixed.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['dtype'], d['ms_per_step'], '%.3g'%d['value'])"
