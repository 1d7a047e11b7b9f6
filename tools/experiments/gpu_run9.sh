timeout 600 python bench.py --no-cpu-baseline --steps 20 --config c2 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_c2.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['config'], d['ms_per_step'], d['value'], d['roofline']['launch_s'], d['launches_per_vcycle'], d['cg'])"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --precision mixed"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:warp_prolongate -s 9 -c 1 -o gpurun_out/prof_prolong_f32 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo full=$?
