#!/bin/bash
# ncu launch list + full captures (edge kernels with source, memory-bound
# kernels for DRAM GB/s) + compute-sanitizer on smoke.  usage: TAG
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02a}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gpu-baseline --e2e-steps 1 --profile-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $B > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_${TAG}.log
for K in k_edge_bwd_fmws k_edge_fwd_ws; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${K}" -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_${K} $B > gpurun_out/ncu_full_${TAG}_${K}.log 2>&1
  echo "full $K exit $?" >> gpurun_out/ncu_full_${TAG}_${K}.log
done
timeout 900 ncu --set full --clock-control none -k "regex:k_scan_rows|k_nbr_assemble|k_noise_baoa_ring|k_forces_finish|k_node_post_pre_tc|k_node_post_readout_tc|k_node_prebwd_postbwd_tc" -s 20 -c 12 \
  -o gpurun_out/prof_${TAG}_small $B > gpurun_out/ncu_full_${TAG}_small.log 2>&1
echo "full small exit $?" >> gpurun_out/ncu_full_${TAG}_small.log
[ -n "$SKIP_SANITIZER" ] || for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 50 python __graft_entry__.py smoke > gpurun_out/sanitizer_${T}.log 2>&1
  echo "sanitizer $T exit $?" >> gpurun_out/sanitizer_${T}.log
done
ls -la gpurun_out
tail -n 3 gpurun_out/sanitizer_*.log
