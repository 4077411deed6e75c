cd "${GRAFT_REPO_ROOT:-/root/repo}"
for tool in memcheck racecheck synccheck initcheck; do
  for case in fused general staged strips fp32 tiles; do  # every kernel family
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    [ $tool = racecheck ] && extra="--racecheck-report hazard"
    out=$(timeout 600 compute-sanitizer --tool $tool $extra python tools/sanitize_case.py --case $case 2>&1 | grep -E "SUMMARY|case ok" | tr '\n' ' ')
    echo "$tool $case: $out"
  done
done
