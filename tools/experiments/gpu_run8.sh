timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
for P in fp64 mixed; do
timeout 600 python bench.py --no-cpu-baseline --steps 30 --precision $P > gpurun_out/bench_$P.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_$P.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['dtype'], d['ms_per_step'], d['value'], d['roofline']['launch_s'], d['roofline']['frac'], d['cg']['iters'])"
done
