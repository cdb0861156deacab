# A/B of the GEMM's L2 policy and raster group on cfg5 fc1 (bench main line only)
mkdir -p gpurun_out/l2ab
for cfg in "0 0" "1 0" "0 0" "1 0" "1 16" "0 0" "1 16"; do
  set -- $cfg
  I8MM_GEMM_L2POL=$1 I8MM_GROUP_M=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-comparators --no-parity --no-peak --e2e-steps 1 > gpurun_out/l2ab/b_$1_$2.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/l2ab/b_$1_$2.json').read().strip().splitlines()[-1]);print('pol',$1,'group',$2,round(d['value'],1),'TOPS',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'],'MHz')"
done
