#!/bin/bash
# GEMM raster A/B (dev tool): GEMM-only time and DRAM bytes per group size.
for g in 1 2 4 8 16 32; do I8MM_GROUP_M=$g timeout 200 python scripts/ab_epi.py gm=$g; done
for g in 1 8 64; do
  I8MM_GROUP_M=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm_i8 -s 10 -c 2 --csv python scripts/ab_epi.py ncu 2>/dev/null | grep -v "^==" | cut -d, -f5,15-16 > gpurun_out/raster_gm$g.csv
done
