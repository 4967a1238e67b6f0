#!/bin/bash
# Round evidence in one call: GPU tests, smoke, bench line, per-kernel bench,
# ncu launch list of the bench command, and one full ncu capture of K3.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
timeout 600 python bench_kernels.py --out gpurun_out/kernels.json > gpurun_out/kernels.log 2>&1; echo "kernels exit $?" >> gpurun_out/kernels.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches exit $?" >> gpurun_out/ncu_launch_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k3_lmhead -s 3 -c 1 \
  -o gpurun_out/k3_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full.log 2>&1; echo "full exit $?" >> gpurun_out/ncu_full.log
for f in pytest_gpu smoke bench bench_ref kernels ncu_launch_bench ncu_full; do echo "== $f"; tail -n 2 gpurun_out/$f.log | cut -c1-400; done
