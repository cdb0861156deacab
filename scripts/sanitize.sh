#!/bin/bash
# compute-sanitizer over scripts/sanitize.py, one tool x stage per process;
# summary lines -> gpurun_out/sanitize/summary.txt
O=gpurun_out/sanitize; mkdir -p $O
: > $O/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  for st in functional module splitk swapab decode peers siblings f32 peak; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py $st > $O/${tool}_${st}.log 2>&1
    rc=$?
    s=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $O/${tool}_${st}.log | tail -1)
    ok=$(grep -c "ALL STAGES OK" $O/${tool}_${st}.log)
    echo "$tool $st rc=$rc ok=$ok :: $s" | tee -a $O/summary.txt
  done
done
