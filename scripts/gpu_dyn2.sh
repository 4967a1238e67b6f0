# Dynamic K3 schedule with and without the die map: steady bench A/B (alternating) and ncu fabric traffic.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2 3; do
  for da in 0 1; do
    MOSAIC_DIE_AWARE=$da timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e > gpurun_out/dyn2_${da}_$i.log 2>&1
    python -c "
import json; l=[x for x in open('gpurun_out/dyn2_${da}_$i.log') if x.startswith('{')][-1]; d=json.loads(l)
print('die_aware=$da', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'], d['config']['k3_schedule'][:30])"
  done
done
for mode in dynamic die; do
  MOSAIC_K3_MODE=$mode timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k3_lmhead -c 2 python scripts/k3_shapes_ncu.py 2>&1 | grep -E "dram__|fabric|duration" | sed "s/^/$mode /"
done
