# DRAM bytes / time of the cfg5 fc1 GEMM per raster group (ncu metrics pass; dev tool)
mkdir -p gpurun_out/rd
for g in 0 2 4 16 32 64; do
  I8MM_GROUP_M=$g timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:gemm_i8 -s 1 -c 1 --csv python scripts/prof_gemm.py ${1:-16384} ${2:-12288} ${3:-49152} 2 > gpurun_out/rd/g$g.csv 2>/dev/null
  echo "group $g"; grep -E "dram__bytes_read|gpu__time|hit_rate|per_second|xbar2l1tex" gpurun_out/rd/g$g.csv | awk -F'","' '{print "  "$(NF-2)" "$(NF-1)" "$NF}'
done
