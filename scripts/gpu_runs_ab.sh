#!/bin/bash
# Runs-mode A path: parity tests, then an alternating same-box A/B of the bench
# (MOSAIC_A_RUNS=1 default vs 0 = every row through K2) and the per-kernel bench.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 \
  -k "gather or runs or batch or variants or fused" > gpurun_out/pytest_runs.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_runs.log
tail -n 3 gpurun_out/pytest_runs.log
for i in 1 2; do
  for r in 1 0; do
    MOSAIC_A_RUNS=$r timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-activation \
      > gpurun_out/ab_runs${r}_$i.log 2>&1
    python -c "
import json,sys; l=[x for x in open('gpurun_out/ab_runs${r}_$i.log') if x.startswith('{')][-1]; d=json.loads(l)
print('runs=$r', round(d['value']), round(d['e2e']['value']), round(d['roofline']['k3_ms'],3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
  done
done
timeout 600 python bench_kernels.py --out gpurun_out/kern_runs.json > /dev/null 2>&1
python -c "
import json; k=json.load(open('gpurun_out/kern_runs.json'))
for n in ['k3_gather_llada','k3_gather_llada_scattered']: print(n, {a:round(k[n][a],3) for a in k[n] if 'ms' in a})
"
