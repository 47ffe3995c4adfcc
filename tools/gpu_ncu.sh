#!/bin/bash
# ncu launch list of one bench step + full-set captures of named kernels.
# usage: tools/gpu_ncu.sh TAG "regex1|regex2" [extra bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r01}; KRE=${2:-k_edge_bwd|k_edge_fwd}; shift 2
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --profile-steps 1 $*"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $B > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KRE}" -s 6 -c 2 \
  -o gpurun_out/prof_${TAG} $B > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full_${TAG}.log
tail -3 gpurun_out/ncu_launch_${TAG}.log gpurun_out/ncu_full_${TAG}.log
ls -la gpurun_out
