# K3 schedule sweep on one box: ncu DRAM bytes of one bench K3 launch + the steady bench per config.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "16 13" "8 13" "12 13" "16 7" "16 19" "24 13"; do
  set -- $cfg
  export MOSAIC_GROUP_M=$1 MOSAIC_K3_TPS=$2
  d=$(timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k3_lmhead -s 3 -c 1 \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-activation 2>&1 | grep -E "dram__bytes_read|hit_rate" | awk '{print $NF$(NF-1)}' | tr '\n' ' ')
  b=$(timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-activation --no-e2e 2>&1 | grep '^{' | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['k3_ms'],3), d['clocks']['sm_mhz'], d['config']['n_splits'])")
  echo "group_m=$1 tps=$2 dram/hit: $d steady: $b"
done
