#!/bin/bash
# Steady-state (4.5 s) sweep of K3 L2 policy x group_m (cta_group 2), plus cuBLAS
# on the identical GEMM shape on the same box for a power/clock reference.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {
  echo "$1" >> gpurun_out/sweep2.log
  env $1 timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e | python -c "import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']; c=d['clocks']; print(f\"  value={d['value']:.0f} k3={r['k3_ms']:.3f} TF={r['achieved']:.0f} frac={r['frac']:.3f} clk={c['sm_mhz']} {c['reasons']}\")" >> gpurun_out/sweep2.log 2>&1
}
for pol in 0 1 2; do for gm in 8 16 32; do run "MOSAIC_L2_POLICY=$pol MOSAIC_GROUP_M=$gm"; done; done
timeout 300 python scripts/cublas_ref.py >> gpurun_out/sweep2.log 2>&1
cat gpurun_out/sweep2.log
