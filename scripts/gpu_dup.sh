#!/bin/bash
# L2-feed power experiment: K3 with every W box loaded twice (MOSAIC_K3_DUP_B=1) vs normal, steady bench.
mkdir -p gpurun_out; : > gpurun_out/dup.log
M="gpu__time_duration.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for rep in 1 2; do for dup in 0 1; do
  MOSAIC_NVCC_DEFINES="MOSAIC_K3_DUP_B=$dup" timeout 300 python -c "from paper_2601_06562_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
  echo "== DUP_B=$dup" >> gpurun_out/dup.log
  if [ $rep = 1 ]; then
  timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|dram__|l1tex__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF)}' >> gpurun_out/dup.log
  fi
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/dup.log 2>&1
done; done
cat gpurun_out/dup.log
