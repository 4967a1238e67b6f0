#!/bin/bash
# Same-box A/B of K3's die-aware schedule: DRAM bytes of one launch (ncu --metrics, 3 alternations)
# and one --set full capture of each.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
: > gpurun_out/die3.log
for i in 1 2 3; do for da in 0 1; do
  echo "== MOSAIC_DIE_AWARE=$da" >> gpurun_out/die3.log
  MOSAIC_DIE_AWARE=$da timeout 300 ncu --metrics $M --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|dram__|sm__)' \
    | awk -F'","' '{print "   " $(NF-3) " " $(NF)}' >> gpurun_out/die3.log
done; done
for da in 0 1; do
  MOSAIC_DIE_AWARE=$da timeout 1200 ncu --set full --clock-control none -k regex:k3_lmhead -s 3 -c 1 \
    -o gpurun_out/k3_full_da$da python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
cat gpurun_out/die3.log
