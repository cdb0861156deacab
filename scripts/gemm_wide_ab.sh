# A/B of the 512-wide pair tile (I8MM_GEMM_WIDE=1) vs 256-wide (=2) on cfg5 fc1 / cfg2 / cfg4 fc1
for wl in cfg5_fc1 cfg2 cfg4_fc1 cfg5_fc2; do
for w in 2 1 2 1; do
  I8MM_GEMM_WIDE=$w timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-comparators --no-peak --e2e-steps 1 > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$wl','wide' if $w==1 else 'narrow',round(d['value'],1),'TOPS',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'],'MHz',d['clocks']['reasons'],'parity',d['parity']['ok'])"
done; done
