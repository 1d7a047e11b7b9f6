# full default bench line (with the CPU baseline) + mixed + c4 + c5 n=1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_default=$?
timeout 900 python bench.py --precision mixed --no-cpu-baseline > gpurun_out/bench_mixed.log 2>&1; echo bench_mixed=$?
timeout 900 python bench.py --config c4 --steps 20 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo bench_c4=$?
timeout 900 python bench.py --config c5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo bench_c5=$?
timeout 900 python bench.py --config c4 --steps 20 --no-cpu-baseline --precision mixed > gpurun_out/bench_c4_mixed.log 2>&1; echo bench_c4m=$?
timeout 900 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench_c2=$?
