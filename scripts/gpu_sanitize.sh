mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 8 python scripts/sanitize_small.py 2>&1 | grep -vE "^=========     (at|by|Host|Saved|Device)" | grep -E "sanitize run ok|ERROR SUMMARY|RACECHECK SUMMARY|Race reported|Error|Invalid" | head -20
done
