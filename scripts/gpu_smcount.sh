#!/bin/bash
# Power-capped SM-count sensitivity of K3: steady bench with the persistent grid capped at N pairs.
mkdir -p gpurun_out; : > gpurun_out/smcount.log
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for n in 0 66 60; do
  echo "== max pairs $n" >> gpurun_out/smcount.log
  MOSAIC_K3_MAX_CLUSTERS=$n timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/smcount.log 2>&1
done; done
cat gpurun_out/smcount.log
