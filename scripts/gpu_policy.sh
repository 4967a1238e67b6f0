#!/bin/bash
# L2 cache-policy A/B for K3 under the die-aware schedule: steady 300-step bench + DRAM bytes of one launch.
mkdir -p gpurun_out; : > gpurun_out/policy.log
M="dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
for rep in 1 2; do for pol in 1 3 0; do
  echo "== MOSAIC_L2_POLICY=$pol" >> gpurun_out/policy.log
  if [ $rep = 1 ]; then
  MOSAIC_L2_POLICY=$pol timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(dram__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF)}' >> gpurun_out/policy.log
  fi
  MOSAIC_L2_POLICY=$pol timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/policy.log 2>&1
done; done
cat gpurun_out/policy.log
