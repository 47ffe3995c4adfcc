#!/bin/bash
# One iteration on the GPU box: gpu tests, a short bench, the phase
# breakdown, and ncu --set full captures of the named kernels (one launch
# each).  usage: tools/gpu_iter.sh TAG "kernA kernB"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-it}; KERNS=${2:-}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 300 python tools/diag_phase.py > gpurun_out/diag_phase_${TAG}.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --profile-steps 1"
for K in $KERNS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${K}" -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_${K} $B > gpurun_out/ncu_full_${TAG}_${K}.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/diag_phase_${TAG}.log
python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}.json'));print('ms/step',d['ms_per_step'],'ns/day',d['value']);print(d['kernel_share'])"
