mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for gm in 16 4 6 8 16; do
  MOSAIC_K10_GROUP_M=$gm timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k10_ \
    python scripts/ncu_targets.py 2>&1 | grep -E "dram__|duration|per_second" | sed "s/^/k10_gm=$gm /"
done
for i in 1 2; do
for gm in 16 6; do
  MOSAIC_K10_GROUP_M=$gm timeout 600 python scripts/k10_sched_ab.py --reps 2 2>&1 | sed "s/^/gm=$gm /"
done
done
