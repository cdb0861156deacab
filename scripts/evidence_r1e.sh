#!/bin/bash
# Round-1 (late) evidence capture on one B200 (dev tool; run under gpurun).
O=gpurun_out/ev8
mkdir -p $O
timeout 120 python scripts/pcie_bw.py > $O/pcie.json 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.csv
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --workload cfg5_fc1 --steps 20 --warmup 3 --e2e-steps 2 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 300 python bench.py --workload cfg3_decode > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-comparators --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 2 -c 2 -o $O/gemm_cfg2 \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-comparators --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"quantize_bulk|outlier_scan|row_scale" -s 3 -c 3 -o $O/prologue_fc2 \
    python scripts/prologue_bench.py fc2 > /dev/null 2>&1
timeout 600 python scripts/decode_sweep.py > $O/decode_default.log 2>&1
I8MM_DECODE_MAX_M=0 timeout 600 python scripts/decode_sweep.py > $O/decode_prefill.log 2>&1
timeout 120 python scripts/prologue_bench.py > $O/prologue.log 2>&1
I8MM_PROLOGUE_1READ=1 timeout 120 python scripts/prologue_bench.py >> $O/prologue.log 2>&1
ls -la $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --steps 30 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err
