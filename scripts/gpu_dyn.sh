# Dynamic K3 unit schedule: parity tests, ncu DRAM per schedule at LLaDA / Dream, kernel A/B, steady bench A/B.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_executor.py -q -x --timeout 600 > gpurun_out/pytest_dyn.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_dyn.log; tail -n 3 gpurun_out/pytest_dyn.log
for mode in static dynamic die; do
  MOSAIC_K3_MODE=$mode timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:k3_lmhead -c 2 python scripts/k3_shapes_ncu.py 2>&1 | grep -E "dram__|duration|hit_rate|per_second|tensor" | sed "s/^/$mode /"
done
timeout 900 python scripts/k3_die_ab.py --reps 3 2>&1 | tee gpurun_out/dyn_kernels.txt
for i in 1 2; do
  for st in 0 1; do
    MOSAIC_K3_STATIC=$st timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e > gpurun_out/dyn_bench_${st}_$i.log 2>&1
    python -c "
import json; l=[x for x in open('gpurun_out/dyn_bench_${st}_$i.log') if x.startswith('{')][-1]; d=json.loads(l)
print('static=$st', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'], d['config']['k3_schedule'][:40])"
  done
done
