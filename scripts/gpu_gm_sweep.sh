mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for gm in 16 8 12 24 32 16; do
  export MOSAIC_GROUP_M=$gm
  d=$(timeout 300 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:k3_lmhead -s 3 -c 1 \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-activation 2>&1 | grep -E "dram__bytes_read" | awk '{print $NF$(NF-1)}')
  b=$(timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e 2>&1 | grep '^{' | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'])")
  echo "group_m=$gm dram=$d steady: $b"
done
