for C in c4 c5; do
timeout 1500 python bench.py --no-cpu-baseline --steps 10 --config $C > gpurun_out/bench_$C.log 2> gpurun_out/bench_$C.err &
PID=$!; PEAK=0
while kill -0 $PID 2>/dev/null; do R=$(ps -o rss= -p $PID 2>/dev/null | tr -d ' '); [ -n "$R" ] && [ "$R" -gt "$PEAK" ] && PEAK=$R; sleep 2; done
wait $PID; echo bench_$C=$? peak_rss_GB=$((PEAK/1048576))
tail -1 gpurun_out/bench_$C.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['config'], d['ms_per_step'], d['value'], d['roofline']['launch_s'], d['roofline']['frac'], d['config']['setup_s'], d['cg'])"
done
free -g | head -2; nproc
