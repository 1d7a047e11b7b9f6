timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu.log
for pdl in 1 0; do
for c in c3 c2; do
GMG_PDL=$pdl timeout 600 python bench.py --no-cpu-baseline --steps 30 --config $c > gpurun_out/bench_${c}_pdl$pdl.log 2>&1
tail -1 gpurun_out/bench_${c}_pdl$pdl.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pdl=$pdl', d['config']['config'], '%.3f'%d['ms_per_step'], '%.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'], d['cg'])"
done
GMG_PDL=$pdl timeout 600 python bench.py --no-cpu-baseline --steps 30 --config c3 --precision mixed > gpurun_out/bench_c3m_pdl$pdl.log 2>&1
tail -1 gpurun_out/bench_c3m_pdl$pdl.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pdl=$pdl mixed', '%.3f'%d['ms_per_step'], '%.3g'%d['value'])"
done
