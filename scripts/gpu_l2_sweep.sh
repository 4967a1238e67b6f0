#!/bin/bash
# K3 with an L2 persisting set-aside (evict_last A operand): DRAM bytes + steady-state clocks.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('l2', p.L2_cache_size)
from paper_2601_06562_b200 import hotpath; print('max persisting', hotpath.l2_persisting_limit(1<<40))" >> gpurun_out/l2.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_miss.sum"
for cfg in "MOSAIC_K3_TPS=13 MOSAIC_GROUP_M=16 MOSAIC_L2_POLICY=1 MOSAIC_L2_PERSIST_MB=0" \
           "MOSAIC_K3_TPS=13 MOSAIC_GROUP_M=16 MOSAIC_L2_POLICY=1 MOSAIC_L2_PERSIST_MB=40" \
           "MOSAIC_K3_TPS=13 MOSAIC_GROUP_M=16 MOSAIC_L2_POLICY=1 MOSAIC_L2_PERSIST_MB=80" \
           "MOSAIC_K3_TPS=13 MOSAIC_GROUP_M=32 MOSAIC_L2_POLICY=1 MOSAIC_L2_PERSIST_MB=80" \
           "MOSAIC_K3_TPS=33 MOSAIC_GROUP_M=16 MOSAIC_L2_POLICY=1 MOSAIC_L2_PERSIST_MB=40" \
           "MOSAIC_K3_TPS=13 MOSAIC_GROUP_M=16 MOSAIC_L2_POLICY=0 MOSAIC_L2_PERSIST_MB=40" \
           "MOSAIC_K3_TPS=13 MOSAIC_GROUP_M=24 MOSAIC_L2_POLICY=1 MOSAIC_L2_PERSIST_MB=60"; do
  echo "== $cfg" >> gpurun_out/l2.log
  env $cfg timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|dram__|lts__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF-2) " " $(NF)}' >> gpurun_out/l2.log
  env $cfg timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} S={d['config']['n_splits']} clk={c['sm_mhz']} {c['reasons']}\")" >> gpurun_out/l2.log 2>&1
done
cat gpurun_out/l2.log
