#!/bin/bash
# K3 segment-major schedule sweep: DRAM bytes per launch (ncu) + steady-state throughput.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MOSAIC_K3_SEG_SPLITS=4 MOSAIC_K3_TPS=8 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "lmhead_stats or full_size or head_step" > gpurun_out/seg_parity.log 2>&1; tail -1 gpurun_out/seg_parity.log > gpurun_out/seg.log
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for cfg in "MOSAIC_K3_TPS=13 MOSAIC_K3_SEG_SPLITS=0" "MOSAIC_K3_TPS=8 MOSAIC_K3_SEG_SPLITS=4" "MOSAIC_K3_TPS=8 MOSAIC_K3_SEG_SPLITS=8" \
           "MOSAIC_K3_TPS=13 MOSAIC_K3_SEG_SPLITS=3" "MOSAIC_K3_TPS=13 MOSAIC_K3_SEG_SPLITS=5" "MOSAIC_K3_TPS=8 MOSAIC_K3_SEG_SPLITS=4 MOSAIC_GROUP_M=8" \
           "MOSAIC_K3_TPS=8 MOSAIC_K3_SEG_SPLITS=4 MOSAIC_GROUP_M=32" "MOSAIC_K3_TPS=8 MOSAIC_K3_SEG_SPLITS=2" "MOSAIC_K3_TPS=13 MOSAIC_K3_SEG_SPLITS=0"; do
  echo "== $cfg" >> gpurun_out/seg.log
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|dram__|lts__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF-2) " " $(NF)}' >> gpurun_out/seg.log
  env $cfg timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} S={d['config']['n_splits']} clk={c['sm_mhz']} {c['reasons']}\")" >> gpurun_out/seg.log 2>&1
done
cat gpurun_out/seg.log
