mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "die or full_size or head or stats" 2>&1 | tail -2
timeout 900 python scripts/k3_die_ab.py --reps 3 2>&1
for i in 1 2; do
  for st in 0 1; do
    MOSAIC_K3_STATIC=$st timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e > gpurun_out/dyn3_${st}_$i.log 2>&1
    python -c "
import json; l=[x for x in open('gpurun_out/dyn3_${st}_$i.log') if x.startswith('{')][-1]; d=json.loads(l)
print('static=$st', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])"
  done
done
