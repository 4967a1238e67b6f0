mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in 0 1; do
  MOSAIC_K3_WAVES=$w MOSAIC_K3_MODE=dynamic timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:k3_lmhead -c 2 python scripts/k3_shapes_ncu.py 2>&1 | grep -E "dram__|duration|hit_rate" | sed "s/^/waves=$w /"
done
for i in 1 2 3; do
  for w in 0 1; do
    MOSAIC_K3_WAVES=$w timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e > gpurun_out/w_${w}_$i.log 2>&1
    python -c "
import json; l=[x for x in open('gpurun_out/w_${w}_$i.log') if x.startswith('{')][-1]; d=json.loads(l)
print('waves=$w', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])"
  done
done
MOSAIC_K3_WAVES=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "full_size or die or head" 2>&1 | tail -2
