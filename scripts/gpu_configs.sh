#!/bin/bash
# Every BASELINE config on the current code (one gpurun call; PREFIX names the outputs):
# GPU tests, configs[0] tiny, configs[2] Dream 128k, configs[3] MoE 64k, the whole LLaDA 32k
# denoising loop, configs[4] context sweep, then the headline bench.
P=${PREFIX:-r02c}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench_tiny.py --out gpurun_out/${P}_tiny_config.json > gpurun_out/tiny.log 2>&1; echo "tiny exit $?" >> gpurun_out/tiny.log
timeout 1200 python bench_dream.py --out gpurun_out/${P}_dream_bench.json > gpurun_out/dream.log 2>&1; echo "dream exit $?" >> gpurun_out/dream.log
timeout 1200 python bench_moe.py --out gpurun_out/${P}_moe_bench.json > gpurun_out/moe.log 2>&1; echo "moe exit $?" >> gpurun_out/moe.log
timeout 1800 python bench_loop.py --out gpurun_out/${P}_loop_llada32k.json > gpurun_out/loop.log 2>&1; echo "loop exit $?" >> gpurun_out/loop.log
timeout 2400 python bench_context.py --out gpurun_out/${P}_context_sweep.json > gpurun_out/context.log 2>&1; echo "context exit $?" >> gpurun_out/context.log
timeout 600 python bench.py > gpurun_out/${P}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${P}_bench.log
for f in pytest_gpu tiny dream moe loop context ${P}_bench; do echo "== $f"; tail -n 2 gpurun_out/$f.log | cut -c1-400; done
