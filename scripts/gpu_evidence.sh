#!/bin/bash
# Round evidence in one gpurun call (PREFIX names the outputs, default r02):
# build, per-kernel bench, the ncu launch list of the bench command, one
# `ncu --set full` capture of K3 inside the bench command (summarised, with
# the DRAM bytes per launch and the code hash written to
# profiles/k3_traffic.json for bench.py), and the SASS proof of tcgen05/TMA.
P=${PREFIX:-r02}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench_kernels.py --out gpurun_out/${P}_kernels.json > gpurun_out/kernels.log 2>&1; echo "kernels exit $?" >> gpurun_out/kernels.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-activation \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches exit $?" >> gpurun_out/ncu_launch_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k3_lmhead -s 3 -c 1 \
  -o gpurun_out/${P}_k3_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-activation \
  > gpurun_out/ncu_full.log 2>&1; echo "full exit $?" >> gpurun_out/ncu_full.log
python scripts/ncu_summary.py gpurun_out/${P}_k3_full.ncu-rep gpurun_out/${P}_k3_full.json --traffic > /dev/null 2>&1
cuobjdump -sass paper_2601_06562_b200/libmosaic_b200.so | grep -E "Function|UTCHMMA|UTCBAR|UTMALDG|LDTM|UTCQMMA" \
  | awk '/Function/{f=$0; n=0} !/Function/{if (n<6) print f" :: "$0; n++}' > gpurun_out/${P}_sass_excerpt.txt
for f in kernels ncu_launch_bench ncu_full; do echo "== $f"; tail -n 2 gpurun_out/$f.log | cut -c1-300; done
