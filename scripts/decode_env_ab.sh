# cfg3 decode step (bench main line, CUDA graph) under env knobs, interleaved (dev tool)
# usage: bash scripts/decode_env_ab.sh "ENV1=a ENV2=b" "ENV1=c" ...
mkdir -p gpurun_out/dab
for rep in 1 2 3; do
  i=0
  for cfg in "$@"; do
    i=$((i+1))
    env $cfg timeout 300 python bench.py --workload cfg3_decode --steps 200 --warmup 20 --no-extras --no-cpu-baseline --no-comparators --no-parity --no-peak --e2e-steps 1 > gpurun_out/dab/b_$i.json 2>gpurun_out/dab/b_$i.err
    python -c "import json;d=json.loads(open('gpurun_out/dab/b_$i.json').read().strip().splitlines()[-1]);print('$cfg', round(d['ms_per_step']*1e3,1),'us/step', d['clocks']['sm_mhz'],'MHz')" || tail -3 gpurun_out/dab/b_$i.err
  done
done
