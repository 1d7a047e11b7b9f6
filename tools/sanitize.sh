#!/bin/bash
# compute-sanitizer over small hot-path runs (tools/sanitize.py) on one B200, under gpurun
# from the repo root: memcheck (out-of-bounds / misaligned accesses, leaks at exit),
# racecheck (shared-memory hazards of the transposition passes), synccheck (barriers).
# Writes gpurun_out/sanitize/*.log; the summaries go to profiles/.
OUT=gpurun_out/sanitize
mkdir -p $OUT
python tools/sanitize.py > $OUT/plain.log 2>&1 || { tail -20 $OUT/plain.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  # cases 0 2 3 4 5: 3D Q2 families, grandfamilies (c5 recipe), 2D, Q1, mixed precision
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py 0 2 3 4 5 > $OUT/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|its rel|done" $OUT/$tool.log | tail -12
done
