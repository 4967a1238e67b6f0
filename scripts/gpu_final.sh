#!/bin/bash
# Final round evidence on the committed code, one gpurun call (PREFIX names the outputs):
# build, GPU tests, smoke, per-kernel bench + ncu launch list + K3 --set full capture + SASS
# (gpu_evidence.sh), ncu of the HBM-bound kernels, sanitizers, every BASELINE config
# (tiny, Dream, MoE, loop, context sweep), the selection-parity record, the reference arm and
# the headline bench (run last, after the K3 capture wrote profiles/k3_traffic.json).
P=${PREFIX:-r02z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${P}_smoke.log
PREFIX=$P bash scripts/gpu_evidence.sh > gpurun_out/${P}_evidence.log 2>&1
cp gpurun_out/k3_traffic.json profiles/k3_traffic.json
timeout 900 ncu --set full --clock-control none -k regex:"k2_|k6_|k9_|k10_|k11_" -o gpurun_out/${P}_hbm -f python scripts/ncu_targets.py > gpurun_out/ncu_hbm.log 2>&1
python scripts/ncu_summary.py gpurun_out/${P}_hbm.ncu-rep gpurun_out/${P}_ncu_hbm_kernels.json > /dev/null 2>&1
python scripts/hbm_summary.py gpurun_out/${P}_ncu_hbm_kernels.json MEASURED_PEAKS.json > gpurun_out/${P}_ncu_hbm_kernels.txt 2>&1
bash scripts/gpu_sanitize.sh > gpurun_out/${P}_sanitizers.txt 2>&1
timeout 600 python bench_tiny.py --out gpurun_out/${P}_tiny_config.json > gpurun_out/tiny.log 2>&1
timeout 1200 python bench_dream.py --out gpurun_out/${P}_dream_bench.json > gpurun_out/dream.log 2>&1
timeout 1200 python bench_moe.py --out gpurun_out/${P}_moe_bench.json > gpurun_out/moe.log 2>&1
timeout 1800 python bench_loop.py --out gpurun_out/${P}_loop_llada32k.json > gpurun_out/loop.log 2>&1
timeout 2400 python bench_context.py --out gpurun_out/${P}_context_sweep.json > gpurun_out/context.log 2>&1
cp gpurun_out/${P}_context_sweep.json profiles/ 2>/dev/null
timeout 1800 python scripts/selection_parity.py --out gpurun_out/${P}_selection_parity.json > gpurun_out/selection.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${P}_bench_reference.log 2>&1
timeout 600 python bench.py > gpurun_out/${P}_bench.log 2>&1
timeout 900 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_bench_300steps.log 2>&1
for f in ${P}_pytest_gpu ${P}_smoke ${P}_evidence tiny dream moe loop context selection ${P}_bench_reference ${P}_bench ${P}_bench_300steps; do
  echo "== $f"; tail -n 2 gpurun_out/$f.log | cut -c1-300; done
cat gpurun_out/${P}_ncu_hbm_kernels.txt; grep -E "==|SUMMARY" gpurun_out/${P}_sanitizers.txt
