timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in c3 c2; do
timeout 600 python bench.py --no-cpu-baseline --steps 30 --config $c > gpurun_out/bench_$c.log 2>&1
tail -1 gpurun_out/bench_$c.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['config'], d['ms_per_step'], '%.3g'%d['value'], r['launch_s'], r['frac'], d['e2e']['value'], d['cg'])"
done
timeout 600 python bench.py --no-cpu-baseline --steps 30 --config c3 --precision mixed > gpurun_out/bench_c3m.log 2>&1
tail -1 gpurun_out/bench_c3m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('mixed', d['ms_per_step'], '%.3g'%d['value'], r['launch_s'], r['frac'], d['cg'])"
