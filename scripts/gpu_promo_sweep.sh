#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second"
for cfg in "MOSAIC_TMA_L2_PROMOTION=3" "MOSAIC_TMA_L2_PROMOTION=2" "MOSAIC_TMA_L2_PROMOTION=0" "MOSAIC_TMA_L2_PROMOTION=3 MOSAIC_L2_POLICY=0"; do
  echo "== $cfg" >> gpurun_out/promo.log
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|dram__|lts__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF-2) " " $(NF)}' >> gpurun_out/promo.log
  env $cfg timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/promo.log 2>&1
done
cat gpurun_out/promo.log
