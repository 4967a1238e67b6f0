mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_moe.py tests/test_gpu_executor.py -q -x --timeout 600 2>&1 | tail -2
timeout 900 python scripts/k10_sched_ab.py --reps 3
for st in 1 0; do
  MOSAIC_K10_STATIC=$st timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k10_ \
    python scripts/ncu_targets.py 2>&1 | grep -E "dram__|duration|per_second" | sed "s/^/k10_static=$st /"
done
