#!/bin/bash
# A/B timing of libfcg.so against libfcg_b.so (bench only, alternating, 3 rounds).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; echo "pytest A exit $?" >> gpurun_out/pytest_ab.log
FCG_LIB_PATH=$PWD/paper_2602_13140_b200/libfcg_b.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/pytest_ab.log 2>&1; echo "pytest B exit $?" >> gpurun_out/pytest_ab.log
for r in 1 2 3; do
  for v in A B; do
    if [ $v = B ]; then export FCG_LIB_PATH=$PWD/paper_2602_13140_b200/libfcg_b.so; else unset FCG_LIB_PATH; fi
    timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['ms_per_step'], {k:round(v,4) for k,v in d['kernel_share'].items() if k.startswith('edge')})"
  done
done
grep -E "exit|passed|failed" gpurun_out/pytest_ab.log
