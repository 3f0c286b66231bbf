#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (every hot-path kernel at small shapes).
# Writes profiles/<round>/sanitize_<tool>.log; run on the GPU box from the repo root.
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
for tool in memcheck initcheck synccheck racecheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 900 compute-sanitizer --tool $tool $extra --target-processes all \
      python tools/sanitize_run.py > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_summary.txt"
  tail -3 "$OUT/sanitize_$tool.log" >> "$OUT/sanitize_summary.txt"
done
