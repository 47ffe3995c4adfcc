#!/bin/bash
# one --set full capture (with source) of the named kernel(s): tools/gpu_ncu_one.sh TAG "k1 k2" [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=$1; KERNS=$2; shift 2
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gpu-baseline --e2e-steps 1 --profile-steps 1 $*"
for K in $KERNS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${K}" -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_${K} $B > gpurun_out/ncu_full_${TAG}_${K}.log 2>&1
  echo "full $K exit $?" >> gpurun_out/ncu_full_${TAG}_${K}.log
done
ls gpurun_out | grep $TAG
