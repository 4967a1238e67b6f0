mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 compute-sanitizer --tool synccheck --print-limit 4 python scripts/sanitize_small.py > gpurun_out/synccheck_full.txt 2>&1
grep -v "^=========     " gpurun_out/synccheck_full.txt | head -40
