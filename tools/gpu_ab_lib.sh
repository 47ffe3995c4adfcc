#!/bin/bash
# Guarded A/B of libfcg.so (A, new) against libfcg_b.so (B): 90 s smoke of A
# first (abort on hang/failure), parity tests on A, alternating benches.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_a.log 2>&1
rc=$?; echo "smoke A exit $rc"; tail -3 gpurun_out/smoke_a.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_physics.py -m gpu -x -q -p no:cacheprovider -rf > gpurun_out/pytest_ab.log 2>&1; echo "pytest A exit $?" >> gpurun_out/pytest_ab.log
tail -4 gpurun_out/pytest_ab.log
for r in 1 2 3; do
  for v in A B; do
    if [ $v = B ]; then export FCG_LIB_PATH=$PWD/paper_2602_13140_b200/libfcg_b.so; else unset FCG_LIB_PATH; fi
    timeout 120 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-gpu-baseline --e2e-steps 2 "$@" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],4), d['gpu_launches']//d['steps'], {k:round(v,4) for k,v in d['kernel_share'].items() if k.startswith('edge')})"
  done
done
