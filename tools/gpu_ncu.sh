#!/bin/bash
# ncu launch list of one bench step + one --set full capture per kernel name.
# usage: tools/gpu_ncu.sh TAG "kernA kernB" [extra bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r01}; KERNS=${2:-k_edge_bwd_tc k_edge_fwd_tc}; shift 2
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-gpu-baseline --e2e-steps 1 --profile-steps 1 $*"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $B > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_${TAG}.log
for K in $KERNS; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${K}" -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_${K} $B > gpurun_out/ncu_full_${TAG}_${K}.log 2>&1
  echo "full $K exit $?" >> gpurun_out/ncu_full_${TAG}_${K}.log
done
ls -la gpurun_out
