#!/bin/bash
# K3 ring depth on the pair path: 6 (default) vs 7 stages (224 KB ring).
mkdir -p gpurun_out
for st in 6 7 6 7; do
  MOSAIC_NVCC_DEFINES="MOSAIC_K3_STAGES2=$st" timeout 300 python -c "from paper_2601_06562_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
  echo "== stages $st" >> gpurun_out/stages.log
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|sm__)' | awk -F'","' '{print "   " $(NF-3) " " $(NF-2) " " $(NF)}' >> gpurun_out/stages.log
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/stages.log 2>&1
done
timeout 300 python -c "from paper_2601_06562_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
cat gpurun_out/stages.log
