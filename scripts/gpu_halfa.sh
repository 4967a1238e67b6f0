#!/bin/bash
# What halving A's L2 feed would buy (MOSAIC_K3_HALF_A=1 skips A loads on odd tiles: timing only,
# results wrong), at 148 SMs and at 132 SMs (the most a cluster-of-4 grid gets on B200).
mkdir -p gpurun_out; : > gpurun_out/halfa.log
M="l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
for half in 0 1; do
  MOSAIC_NVCC_DEFINES="MOSAIC_K3_HALF_A=$half" timeout 300 python -c "from paper_2601_06562_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
  echo "== HALF_A=$half" >> gpurun_out/halfa.log
  timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(dram__|l1tex__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF)}' >> gpurun_out/halfa.log
  for rep in 1 2; do for n in 0 66; do
    echo "   pairs=$n" >> gpurun_out/halfa.log
    MOSAIC_K3_MAX_CLUSTERS=$n timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/halfa.log 2>&1
  done; done
done
cat gpurun_out/halfa.log
