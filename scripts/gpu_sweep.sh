#!/bin/bash
# K3 schedule sweep: cta_group x group_m on the bench workload (no CPU leg).
mkdir -p gpurun_out
for cg in 2 1; do
  for gm in 4 8 16 32; do
    echo "cg=$cg gm=$gm" >> gpurun_out/sweep.log
    MOSAIC_CTA_GROUP=$cg MOSAIC_GROUP_M=$gm timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
      2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(f\"  value={d['value']:.0f} ms={d['ms_per_step']:.3f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} frac={r['frac']:.3f} clk={d['clocks']['sm_mhz']} reasons={d['clocks']['reasons']}\")
    else: print('  ', l.strip()[:300])" >> gpurun_out/sweep.log
  done
done
cat gpurun_out/sweep.log
