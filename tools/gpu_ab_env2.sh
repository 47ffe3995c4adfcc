#!/bin/bash
# Quick parity + env A/B: tools/gpu_ab_env2.sh "ENV_A" "ENV_B" [bench args]
# e.g. tools/gpu_ab_env2.sh "FCG_BWD_FM=0" "FCG_BWD_FM=1"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
A=$1; B=$2; shift 2
mkdir -p gpurun_out
env $B timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -rf > gpurun_out/pytest_ab.log 2>&1; echo "pytest B exit $?" >> gpurun_out/pytest_ab.log
tail -3 gpurun_out/pytest_ab.log
for r in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then E=$A; else E=$B; fi
    env $E timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-gpu-baseline --e2e-steps 2 "$@" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['kernel_share'].items() if k.startswith('edge')}, round(d['roofline']['avg_launch_ms'],4))"
  done
done
