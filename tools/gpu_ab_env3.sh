#!/bin/bash
# Guarded env A/B: a 90 s smoke of B first (abort on hang/failure), then
# parity tests on B and alternating bench runs.  usage: ENV_A ENV_B [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
A=$1; B=$2; shift 2
mkdir -p gpurun_out
env $B timeout 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_b.log 2>&1
rc=$?; echo "smoke B exit $rc"; tail -2 gpurun_out/smoke_b.log
if [ $rc -ne 0 ]; then exit 1; fi
env $B timeout 500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -rf > gpurun_out/pytest_ab.log 2>&1; echo "pytest B exit $?" >> gpurun_out/pytest_ab.log
tail -3 gpurun_out/pytest_ab.log
for r in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then E=$A; else E=$B; fi
    env $E timeout 120 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-gpu-baseline --e2e-steps 2 "$@" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['kernel_share'].items() if k.startswith('edge')}, round(d['roofline']['avg_launch_ms'],4))"
  done
done
