#!/bin/bash
# Round-1 evidence capture on one B200 (dev tool; run under gpurun).
set -x
O=gpurun_out/ev
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.csv
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-comparators --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 4 -c 2 -o $O/gemm_cfg2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-comparators --e2e-steps 1 > /dev/null 2>&1
timeout 300 python scripts/decode_sweep.py > $O/decode_default.log 2>&1
I8MM_DECODE_MAX_M=0 timeout 300 python scripts/decode_sweep.py > $O/decode_prefill.log 2>&1
I8MM_DECODE_MAX_M=16 timeout 300 ncu --set full --clock-control none -k regex:decode -s 2 -c 1 -o $O/decode_fc1_m1 \
    python scripts/decode_sweep.py fc1 1 > /dev/null 2>&1
for c in "qkvo 1" "fc1 1" "fc2 16"; do echo "== $c"; timeout 120 python scripts/decode_timeline.py $c; done > $O/decode_timeline.log 2>&1
ls -la $O
