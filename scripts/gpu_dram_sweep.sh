#!/bin/bash
# DRAM bytes / L2 hit rate of K3 per schedule config (one ncu pass per config).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second"
for cfg in "MOSAIC_CTA_GROUP=2 MOSAIC_L2_POLICY=0 MOSAIC_GROUP_M=8" "MOSAIC_CTA_GROUP=2 MOSAIC_L2_POLICY=0 MOSAIC_GROUP_M=16" \
           "MOSAIC_CTA_GROUP=2 MOSAIC_L2_POLICY=0 MOSAIC_GROUP_M=32" "MOSAIC_CTA_GROUP=2 MOSAIC_L2_POLICY=1 MOSAIC_GROUP_M=16" \
           "MOSAIC_CTA_GROUP=2 MOSAIC_L2_POLICY=2 MOSAIC_GROUP_M=16" "MOSAIC_CTA_GROUP=2 MOSAIC_L2_POLICY=0 MOSAIC_GROUP_M=64" \
           "MOSAIC_CTA_GROUP=1 MOSAIC_L2_POLICY=0 MOSAIC_GROUP_M=16" "MOSAIC_CTA_GROUP=1 MOSAIC_L2_POLICY=0 MOSAIC_GROUP_M=32"; do
  echo "== $cfg" >> gpurun_out/dram.log
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|dram__|lts__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF-2) " " $(NF)}' >> gpurun_out/dram.log
done
cat gpurun_out/dram.log
