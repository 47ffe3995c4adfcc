#!/bin/bash
# tests + smoke + bench, then ncu captures of the named kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-run}; KERNS=${2:-}
bash tools/gpu_check.sh
if [ -n "$KERNS" ]; then bash tools/gpu_ncu.sh "$TAG" "$KERNS" > /dev/null 2>&1; fi
ls gpurun_out
