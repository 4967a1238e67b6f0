#!/bin/bash
# Pre-tiled W experiment (MOSAIC_K3_WBLOCKED=1: each W TMA box one contiguous 32 KB block):
# parity hash, DRAM bytes, steady throughput; alternating with the row-major layout on one box.
mkdir -p gpurun_out; : > gpurun_out/wblocked.log
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for wb in 0 1; do MOSAIC_K3_WBLOCKED=$wb timeout 120 python scratch/wblocked_check.py >> gpurun_out/wblocked.log 2>&1; done
M="dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second"
for rep in 1 2; do for wb in 0 1; do
  echo "== WBLOCKED=$wb" >> gpurun_out/wblocked.log
  if [ $rep = 1 ]; then
  MOSAIC_K3_WBLOCKED=$wb timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(dram__|gpu__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF)}' >> gpurun_out/wblocked.log
  fi
  MOSAIC_K3_WBLOCKED=$wb timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/wblocked.log 2>&1
done; done
cat gpurun_out/wblocked.log
