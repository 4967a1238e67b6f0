#!/bin/bash
# Die-aware K3 schedule vs default with the full-flush die probe (clean map): ncu DRAM/clock of one
# launch + a 300-step steady bench per config, alternating configs to expose box drift.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "
import torch; from paper_2601_06562_b200 import hotpath, _native; _native.load()
t, info = hotpath.die_map(torch.device('cuda', 0)); print(info); print(''.join(str(int(v)) for v in t.cpu()))" > gpurun_out/die2.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_ltcfabric.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for cfg in "MOSAIC_DIE_AWARE=0" "MOSAIC_DIE_AWARE=1" "MOSAIC_DIE_AWARE=0" "MOSAIC_DIE_AWARE=1" "MOSAIC_DIE_AWARE=1 MOSAIC_GROUP_M=12"; do
  echo "== $cfg" >> gpurun_out/die2.log
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|dram__|lts__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF)}' >> gpurun_out/die2.log
  env $cfg timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/die2.log 2>&1
done
cat gpurun_out/die2.log
