# GEMM launches chunked by raster groups (default) vs one launch (I8MM_GEMM_CHUNK_WAVES=0),
# bench lines of every prefill workload, interleaved (dev tool)
for rep in 1 2; do for cw in 0 8; do for wl in cfg5_fc1 cfg5_fc2 cfg2 cfg4_fc1; do
  I8MM_GEMM_CHUNK_WAVES=$cw timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-comparators --no-parity --no-peak --e2e-steps 1 > gpurun_out/gc.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/gc.json').read().strip().splitlines()[-1]);print('$wl waves $cw',round(d['value'],1),'TOPS',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'],'MHz',d['clocks']['reasons'])"
done; done; done
