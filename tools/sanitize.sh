# compute-sanitizer over small corrections (SURVEY §4.3 layer 5): memcheck,
# racecheck (shared memory), synccheck, initcheck on C1, a 64^3 C2 crop, the
# 2D C4 crop, a C3 crop, the sharded loopback, the host entry and the Theorem 1 /
# edit-log entry points (tools/san_case.py)
out=gpurun_out/sanitize
mkdir -p $out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 100000 python tools/san_case.py > $out/$tool.log 2>&1
  echo "$tool: exit $? ; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/$tool.log | tail -1)"
done
