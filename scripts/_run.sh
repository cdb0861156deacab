O=gpurun_out/pdl
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-comparators --e2e-steps 2 > $O/bench_pdl_$i.json 2> $O/bench.err
I8MM_PDL=0 timeout 300 python bench.py --no-cpu-baseline --no-comparators --e2e-steps 2 > $O/bench_nopdl_$i.json 2>> $O/bench.err
done
timeout 120 python scripts/prologue_bench.py > $O/pro.log 2>&1
I8MM_PDL=0 timeout 120 python scripts/prologue_bench.py >> $O/pro.log 2>&1
