#!/bin/bash
# Bench-only A/B of libfcg.so (A) against libfcg_b.so (B) for performance
# probes whose numerics are not final (no smoke / parity gate): three
# alternating pairs.  Bench-arg pass-through: tools/gpu_ab_bench.sh [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for r in ${AB_PAIRS:-1 2 3}; do
  for v in A B; do
    if [ $v = B ]; then export FCG_LIB_PATH=$PWD/paper_2602_13140_b200/libfcg_b.so; else unset FCG_LIB_PATH; fi
    timeout 120 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-gpu-baseline --e2e-steps 2 "$@" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],4), d['gpu_launches']//d['steps'], {k:round(v,4) for k,v in d['kernel_share'].items() if k.startswith('edge')})"
  done
done
