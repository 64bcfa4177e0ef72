# compute-sanitizer evidence: every kernel family (tools/sanitize_cases.py) under each tool
mkdir -p gpurun_out
timeout 300 python tools/sanitize_cases.py > gpurun_out/sanit_plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/sanit_plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanit_$t.log 2>&1
  echo "== $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanit_$t.log | tr '\n' ' ')"
done
