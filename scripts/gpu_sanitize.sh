# compute-sanitizer over every kernel family (scripts/sanitize_small.py). Only this
# library's kernels are checked (mangled names contain "mosaic"): cuDNN's SDPA
# kernel, which smoke()'s tiny model step launches, trips synccheck's "Missing
# init" on its own mbarriers.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --kernel-name regex=mosaic --print-limit 8 python scripts/sanitize_small.py 2>&1 \
    | grep -vE "^=========     (at|by|Host|Saved|Device)" \
    | grep -iE "sanitize run ok|ERROR SUMMARY|RACECHECK SUMMARY|Race reported|error|Invalid" | head -20
done
