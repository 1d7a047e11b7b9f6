timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 --config c2 > gpurun_out/bench_c2.log 2>&1
tail -1 gpurun_out/bench_c2.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['config'], d['ms_per_step'], '%.3g'%d['value'], d['cg'])"
