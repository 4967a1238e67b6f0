mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2 3; do
 for da in 0 1; do
  MOSAIC_DIE_AWARE=$da timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-activation 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print('da=$da', 'steps=20', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])"
 done
done
for da in 0 1 0 1; do
  MOSAIC_DIE_AWARE=$da timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e --no-activation 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print('da=$da', 'steps=300', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])"
done
timeout 600 python bench_kernels.py --out gpurun_out/kern_b.json > /dev/null 2>&1
python -c "
import json; k=json.load(open('gpurun_out/kern_b.json'))
for n in ['k3_gather_llada','k3_gather_llada_scattered','k3_lmhead_llada','k3_lmhead_dream','k3_lmhead_moe','k3_lmhead_llada_shard8']: print(n, {a:round(k[n][a],3) for a in k[n] if 'ms' in a})
"
