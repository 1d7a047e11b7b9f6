# round-1 refresh: ncu --set full of the plain operator kernel (the one bench.py's
# roofline times) in both precisions, launch lists of one V-cycle, bench lines.
for P in fp64 mixed; do
  if [ $P = fp64 ]; then KN="fam_tensor_apply<.int.2, double, .int.0>"; else KN="fam_tensor_apply<.int.2, float, .int.0>"; fi
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile --precision $P"
  $CMD > gpurun_out/plain_$P.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      --kernel-name-base demangled -k "regex:$KN" -c 1 -o gpurun_out/prof_apply0_$P -f $CMD > gpurun_out/ncu_full_$P.log 2>&1
  echo full_$P=$?
  [ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/launches_$P.csv $CMD > gpurun_out/ncu_launches_$P.log 2>&1
  echo launches_$P=$?
done
