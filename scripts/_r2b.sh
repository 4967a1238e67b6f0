mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "gather" > gpurun_out/pytest_g.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_g.log
tail -n 2 gpurun_out/pytest_g.log
timeout 600 python bench_kernels.py --out gpurun_out/kern_b.json > /dev/null 2>&1
python -c "
import json; k=json.load(open('gpurun_out/kern_b.json'))
for n in ['k3_gather_llada','k3_gather_llada_scattered','k3_lmhead_llada']: print(n, {a:round(k[n][a],3) for a in k[n] if 'ms' in a})
"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k3_lmhead -s 2 -c 2 python scripts/_k3_ab.py 2>&1 | grep -E "k3_lmhead|duration|tensor|inst_exec|per_second"
