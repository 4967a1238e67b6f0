mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python scripts/k3_die_ab.py > gpurun_out/r02d_k3_die_ab.txt 2>&1
cat gpurun_out/r02d_k3_die_ab.txt
bash scripts/gpu_sanitize.sh > gpurun_out/r02d_sanitizers.txt 2>&1
cat gpurun_out/r02d_sanitizers.txt
