# the plain level operator (finest level, fp64) under ncu with its default clock control (locked base clocks)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active \
    --profile-from-start off --kernel-name-base demangled -k "regex:fam_tensor_apply<.int.2, double, .int.0>" -c 1 --csv \
    --log-file gpurun_out/ncu_clk_base.csv $CMD > gpurun_out/ncu_clk_base.log 2>&1
echo base=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active \
    --clock-control none --profile-from-start off --kernel-name-base demangled -k "regex:fam_tensor_apply<.int.2, double, .int.0>" -c 1 --csv \
    --log-file gpurun_out/ncu_clk_none.csv $CMD > gpurun_out/ncu_clk_none.log 2>&1
echo none=$?
