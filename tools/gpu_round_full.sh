#!/bin/bash
# One refresh of every round artefact at HEAD (tag $1): full -m gpu suite,
# parity margins + bench lines of every quoted config + launch list
# (gpu_round2b.sh), ncu captures (gpu_prof_r02.sh, without its sanitizer
# pass), compute-sanitizer (gpu_sanitize.sh), the reference arm.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02k}
mkdir -p gpurun_out
nproc > gpurun_out/nproc_$TAG.txt
bash tools/gpu_tests.sh > gpurun_out/gpu_tests_$TAG.out 2>&1
cp gpurun_out/pytest_gpu.log gpurun_out/pytest_gpu_$TAG.log
bash tools/gpu_round2b.sh $TAG > gpurun_out/round2b_$TAG.log 2>&1
SKIP_SANITIZER=1 bash tools/gpu_prof_r02.sh $TAG > gpurun_out/prof_$TAG.log 2>&1
bash tools/gpu_sanitize.sh > gpurun_out/sanitize_$TAG.log 2>&1
timeout 900 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_$TAG/bench_ref_arm.json 2> gpurun_out/bench_ref_$TAG.err
echo "ref exit $?" >> gpurun_out/bench_ref_$TAG.err
tail -3 gpurun_out/pytest_gpu_$TAG.log
tail -9 gpurun_out/round2b_$TAG.log
tail -n 2 gpurun_out/sanitizer_*.log
tail -c 600 gpurun_out/bench_$TAG/bench_ref_arm.json
