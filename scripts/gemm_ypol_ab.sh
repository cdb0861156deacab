# cfg5 fc1 GEMM under L2 policy bits (I8MM_GEMM_L2POL: 1 A evict_last, 2 B evict_first, 4 Y stores evict_first):
# one ncu metrics pass (DRAM bytes, time, clock) and the bench main line per setting (dev tool)
mkdir -p gpurun_out/ypol
for pol in 0 4 5 6 7; do
  I8MM_GEMM_L2POL=$pol timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_i8 -s 1 -c 1 --csv python scripts/prof_gemm.py 16384 12288 49152 2 > gpurun_out/ypol/n$pol.csv 2>/dev/null
  echo "pol $pol: $(grep -E 'dram__bytes_read|dram__bytes_write|gpu__time|hit_rate|per_second' gpurun_out/ypol/n$pol.csv | awk -F'","' '{printf "%s=%s %s  ", $(NF-2), $NF, $(NF-1)}' | sed 's/"//g')"
done
for rep in 1 2; do for pol in 0 4 5; do
  I8MM_GEMM_L2POL=$pol timeout 600 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-comparators --no-parity --no-peak --e2e-steps 1 > gpurun_out/ypol/b$pol.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ypol/b$pol.json').read().strip().splitlines()[-1]);print('bench pol',$pol,round(d['value'],1),'TOPS',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'],'MHz',d['clocks']['reasons'])"
done; done
