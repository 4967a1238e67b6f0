#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 1200 python bench_moe.py --out gpurun_out/moe_bench.json > gpurun_out/bench_moe.log 2>&1; echo "bench_moe exit $?" >> gpurun_out/bench_moe.log
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/bench.log; tail -n 5 gpurun_out/bench_moe.log
