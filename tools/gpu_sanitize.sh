#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over smoke(): tools/gpu_sanitize.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 50 --target-processes all \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_${T}.log 2>&1
  echo "sanitizer $T exit $?" >> gpurun_out/sanitizer_${T}.log
done
tail -n 4 gpurun_out/sanitizer_*.log
