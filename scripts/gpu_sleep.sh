#!/bin/bash
# K3 poll backoff (epilogue / producer nanosleep) vs steady-state clocks and throughput.
mkdir -p gpurun_out
for defs in "" "MOSAIC_K3_EPI_SLEEP_NS=256" "MOSAIC_K3_EPI_SLEEP_NS=1000" "MOSAIC_K3_EPI_SLEEP_NS=256 MOSAIC_K3_PROD_SLEEP_NS=64" "MOSAIC_K3_EPI_SLEEP_NS=1000 MOSAIC_K3_PROD_SLEEP_NS=128" ""; do
  MOSAIC_NVCC_DEFINES="$defs" timeout 300 python -c "from paper_2601_06562_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
  echo "== [$defs]" >> gpurun_out/sleep.log
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k3_lmhead -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(gpu__|sm__)' | awk -F'","' '{print "   " $(NF-3) " " $(NF-2) " " $(NF)}' >> gpurun_out/sleep.log
  for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"   steady value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} clk={c['sm_mhz']}\")" >> gpurun_out/sleep.log 2>&1
  done
done
timeout 300 python -c "from paper_2601_06562_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "lmhead_stats or head_step" 2>&1 | tail -1 >> gpurun_out/sleep.log
cat gpurun_out/sleep.log
