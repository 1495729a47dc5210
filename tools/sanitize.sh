#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tests/sanitize_target.py (GPU box).
# Summaries in gpurun_out/sanitizer_*.log; copy the summary into profiles/ after review.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_target.py ${KINDS:-} > gpurun_out/sanitizer_$tool.log 2>&1
  echo "exit $?"
  grep -E "ok|done|ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/sanitizer_$tool.log | head -30
done
