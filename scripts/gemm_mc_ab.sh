# A/B of the GEMM's B-multicast cluster (MC=2) vs plain CTA pairs, cfg5 fc1 + cfg2 (bench main line only)
for wl in cfg5_fc1 cfg2; do
for mc in 1 2 1 2 1 2; do
  I8MM_GEMM_MC=$mc timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-comparators --no-parity --no-peak --e2e-steps 1 > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$wl','mc',$mc,round(d['value'],1),'TOPS',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'],'MHz',d['clocks']['reasons'])"
done; done
