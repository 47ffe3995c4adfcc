#!/bin/bash
# A/B of one library with and without an environment setting (B = with it).
# usage: tools/gpu_ab_env.sh FCG_PDL=0 [bench args...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
SET=$1; shift
ARGS=${*:-"--steps 100 --warmup 10"}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; echo "pytest A exit $?" >> gpurun_out/pytest_ab.log
env $SET timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/pytest_ab.log 2>&1; echo "pytest B exit $?" >> gpurun_out/pytest_ab.log
for r in 1 2 3; do
  for v in A B; do
    E=""; [ $v = B ] && E=$SET
    env $E timeout 300 python bench.py $ARGS --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['ms_per_step'], d['value'], d['e2e']['value'])"
  done
done
grep -E "exit|passed|failed" gpurun_out/pytest_ab.log
