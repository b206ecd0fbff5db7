#!/bin/bash
# compute-sanitizer over every kernel of the library: memcheck,
# racecheck (shared-memory hazards: the TMA / mbarrier rings, block reductions),
# synccheck (barriers), initcheck (reads of uninitialised device memory).
# Logs: gpurun_out/r2_sanitizer_<tool>.log
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  args=""
  [ "$tool" = "memcheck" ] && args="--sym"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 \
      python measure/sanitize_driver.py $args > gpurun_out/r2_sanitizer_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r2_sanitizer_$tool.log | tail -1)"
done
