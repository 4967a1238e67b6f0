#!/bin/bash
# Run-to-run spread of the default bench line and one long steady run (same box).
mkdir -p gpurun_out; : > gpurun_out/repeat.log
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2 3 4 5; do
  timeout 300 python bench.py --no-cpu-baseline | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; e=d['e2e']; print(f\"default run $i: value={d['value']:.0f} e2e={e['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']} reasons={c['reasons']}\")" >> gpurun_out/repeat.log 2>&1
done
timeout 600 python bench.py --steps 3000 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"3000 steps: value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']} samples={c['samples']} reasons={c['reasons']}\")" >> gpurun_out/repeat.log 2>&1
nvidia-smi --query-gpu=name,power.limit,temperature.gpu,clocks.max.sm --format=csv >> gpurun_out/repeat.log
cat gpurun_out/repeat.log
