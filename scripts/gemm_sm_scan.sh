# cfg5 fc1 GEMM time vs number of CTA-pair clusters (L2-bound test)
for c in 74 64 56 48 74 40; do
  I8MM_GEMM_MAX_CLUSTERS=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-comparators --no-parity --no-peak --e2e-steps 1 > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('clusters',$c,round(d['value'],1),'TOPS',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'],'MHz',d['clocks']['reasons'])"
done
