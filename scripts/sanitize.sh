#!/bin/bash
# compute-sanitizer over scripts/sanitize_case.py; logs to gpurun_out/${TAG}_sanitizer_<tool>.log
O=gpurun_out; T=${TAG:-san}
for tool in ${TOOLS:-memcheck synccheck racecheck initcheck}; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --kernel-name-exclude kns=at:: python scripts/sanitize_case.py > $O/${T}_sanitizer_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok' $O/${T}_sanitizer_$tool.log | tr '\n' ' ')"
done
