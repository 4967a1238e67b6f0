#!/bin/bash
# ncu evidence for the step: (1) launch list with per-launch device time,
# (2) one full-set capture of the K3 LM-head kernel (top kernel).
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_bench.log 2>&1
echo "launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k3_lmhead -s 3 -c 1 \
  -o gpurun_out/k3_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full.log 2>&1
echo "full exit $?"
ls -la gpurun_out
