#!/bin/bash
# cg2 evidence: launch list, full ncu capture of K3, and long (steady-state) benches cg1 vs cg2.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k3_lmhead -s 3 -c 1 \
  -o gpurun_out/k3_cg2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full.log 2>&1
for rep in 1 2; do
  for cg in 2 1; do
    echo "cg=$cg rep=$rep" >> gpurun_out/long.log
    MOSAIC_CTA_GROUP=$cg timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; print(f\"  value={d['value']:.0f} ms={d['ms_per_step']:.3f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} frac={r['frac']:.3f} clk={d['clocks']}\")" >> gpurun_out/long.log 2>&1
  done
done
cat gpurun_out/long.log
