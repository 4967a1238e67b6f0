# Die-aware vs default K3 unit schedule: kernel bursts at every strong-scaling shape, the
# steady bench (alternating), and ncu DRAM bytes of one bench K3 launch per schedule.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python scripts/k3_die_ab.py --reps 4 > gpurun_out/die_ab_kernels.txt 2>&1
cat gpurun_out/die_ab_kernels.txt
for i in 1 2; do
  for da in 1 0; do
    MOSAIC_DIE_AWARE=$da timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e \
      > gpurun_out/die_ab_bench_${da}_$i.log 2>&1
    python -c "
import json; l=[x for x in open('gpurun_out/die_ab_bench_${da}_$i.log') if x.startswith('{')][-1]; d=json.loads(l)
print('die_aware=$da', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'], d['config']['k3_schedule'])"
  done
done
for da in 1 0; do
  MOSAIC_DIE_AWARE=$da timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:k3_lmhead -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-activation 2>&1 \
    | grep -E "k3_lmhead|dram__|duration|hit_rate|per_second" | sed "s/^/die_aware=$da /"
done
