#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/pytest_sharded.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_sharded.log
timeout 600 python bench.py --steps 200 --warmup 20 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "bench exit $?" >> gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref exit $?" >> gpurun_out/bench_ref.err
tail -5 gpurun_out/pytest_sharded.log; tail -2 gpurun_out/bench_c2.err gpurun_out/bench_ref.err
