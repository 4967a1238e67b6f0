#!/bin/bash
# Round-2 design experiments, one gpurun call each: bash scripts/gpu_experiments.sh NAME
# (the profiles/r02*_*.txt records name the experiment that produced them). All alternate
# their arms on one box; numbers printed to stdout.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
case "$1" in
runs_ab)
# Runs-mode A path: parity tests, then an alternating same-box A/B of the bench
# (MOSAIC_A_RUNS=1 default vs 0 = every row through K2) and the per-kernel bench.
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
;;
die_ab)
# Die-aware vs default K3 unit schedule: kernel bursts at every strong-scaling shape, the
# steady bench (alternating), and ncu DRAM bytes of one bench K3 launch per schedule.
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
;;
dyn)
# Dynamic K3 unit schedule: parity tests, ncu DRAM per schedule at LLaDA / Dream, kernel A/B, steady bench A/B.
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
;;
dyn_die)
# Dynamic K3 schedule with and without the die map: steady bench A/B (alternating) and ncu fabric traffic.
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
;;
dyn_claim)
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
;;
sched_sweep)
# K3 schedule sweep on one box: ncu DRAM bytes of one bench K3 launch + the steady bench per config.
for cfg in "16 13" "8 13" "12 13" "16 7" "16 19" "24 13"; do
  set -- $cfg
  export MOSAIC_GROUP_M=$1 MOSAIC_K3_TPS=$2
  d=$(timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k3_lmhead -s 3 -c 1 \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-activation 2>&1 | grep -E "dram__bytes_read|hit_rate" | awk '{print $NF$(NF-1)}' | tr '\n' ' ')
  b=$(timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e 2>&1 | grep '^{' | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'], d['config']['n_splits'])")
  echo "group_m=$1 tps=$2 dram/hit: $d steady: $b"
done
;;
gm_sweep)
for gm in 16 8 12 24 32 16; do
  export MOSAIC_GROUP_M=$gm
  d=$(timeout 300 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:k3_lmhead -s 3 -c 1 \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-activation 2>&1 | grep -E "dram__bytes_read" | awk '{print $NF$(NF-1)}')
  b=$(timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e 2>&1 | grep '^{' | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])")
  echo "group_m=$gm dram=$d steady: $b"
done
;;
k10_dyn)
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_moe.py tests/test_gpu_executor.py -q -x --timeout 600 2>&1 | tail -2
timeout 900 python scripts/k10_sched_ab.py --reps 3
for st in 1 0; do
  MOSAIC_K10_STATIC=$st timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k10_ \
    python scripts/ncu_targets.py 2>&1 | grep -E "dram__|duration|per_second" | sed "s/^/k10_static=$st /"
done
;;
k10_gm)
for gm in 16 4 6 8 16; do
  MOSAIC_K10_GROUP_M=$gm timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k10_ \
    python scripts/ncu_targets.py 2>&1 | grep -E "dram__|duration|per_second" | sed "s/^/k10_gm=$gm /"
done
for i in 1 2; do
for gm in 16 6; do
  MOSAIC_K10_GROUP_M=$gm timeout 600 python scripts/k10_sched_ab.py --reps 2 2>&1 | sed "s/^/gm=$gm /"
done
done
;;
half_a)
# Halved-A-feed emulation vs the product, 148 SMs and 132 SMs (MOSAIC_K3_MAX_CLUSTERS=66), steady bench, alternating.
R=$(pwd)
rm -rf /tmp/exp && cp -r "$R" /tmp/exp && rm -f /tmp/exp/paper_2601_06562_b200/libmosaic_b200.so
python scripts/exp_half_a.py /tmp/exp/paper_2601_06562_b200/csrc/lmhead.cu
(cd /tmp/exp && timeout 300 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1) || echo "exp build failed"
timeout 300 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  for mc in 0 66; do
    for v in prod half; do
      d=$R; [ $v = half ] && d=/tmp/exp
      (cd $d && MOSAIC_K3_MAX_CLUSTERS=$mc timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e 2>/dev/null | grep '^{' | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v clusters=$mc', round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])")
    done
  done
done
;;
l2_policy)
# K3's L2 policy of the (A, B) loads under the dynamic schedule (MOSAIC_L2_POLICY 0-3): ncu DRAM of
# one bench launch and the 100-step steady bench per policy.
for pol in 1 0 2 3 1; do
export MOSAIC_L2_POLICY=$pol
d=$(timeout 300 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:k3_lmhead -s 3 -c 1 \
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-activation 2>&1 | grep -E "dram__bytes_read" | awk '{print $NF$(NF-1)}')
b=$(timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e 2>&1 | grep '^{' | tail -1 | \
python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])")
echo "policy=$pol dram=$d steady: $b"
done
;;
l2_ab)
# policy 1 vs 3 alternating (steady bench, 100 steps), then the K3 burst at every shape per policy
for i in 1 2 3; do
for pol in 1 3; do
b=$(MOSAIC_L2_POLICY=$pol timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e 2>&1 | grep '^{' | tail -1 | \
python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])")
echo "policy=$pol steady: $b"
done
done
for pol in 1 3; do MOSAIC_L2_POLICY=$pol timeout 900 python scripts/k3_die_ab.py --reps 2 2>&1 | sed "s/^/policy=$pol /"; done
;;
k10_policy)
# K10 weight-tile L2 policy (MOSAIC_K10_B_EVICT_FIRST), ncu per launch on the LLaDA chunk, alternating
for i in 1 2; do
for bf in 0 1; do
MOSAIC_K10_B_EVICT_FIRST=$bf timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k10_ \
python scripts/ncu_targets.py 2>&1 | grep -E "dram__|duration|per_second" | sed "s/^/k10_b_evict_first=$bf /"
done
done
;;
k3_knobs)
# K3 knob sweep under the current defaults: steady bench (100 steps) per setting, each beside a baseline run
for kv in "MOSAIC_K3_TPS=10" "MOSAIC_K3_TPS=16" "MOSAIC_K3_TPS=19" "MOSAIC_K3_TPS=26" "MOSAIC_TMA_L2_PROMOTION=0" "MOSAIC_TMA_L2_PROMOTION=3" "MOSAIC_GROUP_M=12"; do
for arm in base "$kv"; do
b=$( ( [ "$arm" != base ] && export $arm; timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e ) 2>&1 | grep '^{' | tail -1 | \
python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'], d['config']['n_splits'])")
echo "$arm steady: $b"
done
done
;;
stages)
# K3 ring depth (compile-time MOSAIC_K3_STAGES2, default 6) on a copy of the tree, steady bench alternating
R=$(pwd)
for st in 5 7; do
rm -rf /tmp/exp$st && cp -r "$R" /tmp/exp$st && rm -f /tmp/exp$st/paper_2601_06562_b200/libmosaic_b200.so
(cd /tmp/exp$st && MOSAIC_NVCC_DEFINES="MOSAIC_K3_STAGES2=$st" timeout 300 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1) || echo "build $st failed"
done
for i in 1 2; do
for v in 6 5 7; do
d=$R; [ $v != 6 ] && d=/tmp/exp$v
b=$( (cd $d && timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e) 2>&1 | grep '^{' | tail -1 | \
python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])")
echo "stages=$v steady: $b"
done
done
;;
*)
echo "usage: $0 runs_ab|die_ab|dyn|dyn_die|dyn_claim|sched_sweep|gm_sweep|k10_dyn|k10_gm|half_a|l2_policy|l2_ab|k10_policy|k3_knobs|stages"; exit 2
;;
esac
