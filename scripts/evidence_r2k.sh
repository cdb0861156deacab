#!/bin/bash
# Round-2 final evidence capture on one B200 (dev tool; run under gpurun).
O=gpurun_out/ev_r2k
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_r2k.csv python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline --no-comparators --no-parity --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 12 -c 6 -o $O/dec_r2k \
    python bench.py --workload cfg3_decode --steps 3 --warmup 3 --no-extras --no-cpu-baseline --no-comparators --no-parity --no-peak --e2e-steps 1 > /dev/null 2>&1
bash scripts/sanitize.sh > /dev/null 2>&1
cp gpurun_out/sanitize/summary.txt $O/sanitize_summary_r2k.txt
ls -la $O
