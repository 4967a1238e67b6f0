#!/bin/bash
# PDL on/off: tiny hot-path graph, 32-position windowed step, batched block decoding, LLaDA bench.
mkdir -p gpurun_out; : > gpurun_out/pdl.log
for pdl in 0 1 0 1; do
  echo "== MOSAIC_PDL=$pdl" >> gpurun_out/pdl.log
  MOSAIC_PDL=$pdl timeout 600 python bench_kernels.py --out gpurun_out/kp.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/kp.json'))
print('   step_tiny', d['step_tiny'], 'block32', d['step_llada_block32']['eager_ms'], d['step_llada_block32']['graph_ms'], 'llada', d['step_llada'])" >> gpurun_out/pdl.log
  MOSAIC_PDL=$pdl timeout 300 python scratch/time_batch.py | grep -E "B=  ( 1|64)" >> gpurun_out/pdl.log
  MOSAIC_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); print('   bench', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/pdl.log
done
cat gpurun_out/pdl.log
