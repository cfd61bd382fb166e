# compute-sanitizer racecheck / synccheck / memcheck over every kernel family
# (tools/sanitize_point.py) at 64^2 M=8, 128^2 M=4 and 512^2 M=8; logs into
# gpurun_out/sanitize_<tool>_<level>_<M>.log.  usage: bash tools/sanitize.sh [tag]
for pt in "4 8" "5 4" "7 8" "6 32"; do
  set -- $pt
  for tool in memcheck synccheck racecheck; do
    log=gpurun_out/sanitize_${tool}_$1_$2.log
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_point.py $1 $2 > $log 2>&1
    echo "$tool $1 $2 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)"
  done
done
