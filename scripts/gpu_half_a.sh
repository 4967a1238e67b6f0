# Halved-A-feed emulation vs the product, 148 SMs and 132 SMs (MOSAIC_K3_MAX_CLUSTERS=66), steady bench, alternating.
mkdir -p gpurun_out
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
