#!/bin/bash
# Refresh the code-hash-bound evidence after a kernel change (PREFIX names the outputs):
# GPU tests, per-kernel bench + ncu launch list + K3 capture (k3_traffic.json), the context
# sweep, then the bench (20 and 300 steps) reading both.
P=${PREFIX:-r02z}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${P}_smoke.log
PREFIX=$P bash scripts/gpu_evidence.sh > gpurun_out/${P}_evidence.log 2>&1
cp gpurun_out/k3_traffic.json profiles/k3_traffic.json
timeout 2400 python bench_context.py --out gpurun_out/${P}_context_sweep.json > gpurun_out/context.log 2>&1
cp gpurun_out/${P}_context_sweep.json profiles/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/${P}_bench.log 2>&1
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_bench_300steps.log 2>&1
for f in ${P}_pytest_gpu ${P}_smoke ${P}_evidence context ${P}_bench ${P}_bench_300steps; do
  echo "== $f"; tail -n 2 gpurun_out/$f.log | cut -c1-300; done
