#!/bin/bash
# parity margins + bench lines of every quoted config + launch list (tag $1)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02c}
mkdir -p gpurun_out/bench_$TAG
rm -f gpurun_out/parity_margins_$TAG.jsonl
FCG_PARITY_LOG=$PWD/gpurun_out/parity_margins_$TAG.jsonl timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_configs_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_configs_$TAG.log
O=gpurun_out/bench_$TAG
timeout 600 python bench.py --steps 500 --warmup 50 > $O/bench_c2_fp32.json 2> $O/c2.err
timeout 600 python bench.py --steps 500 --warmup 50 --config w16 --no-cpu-baseline > $O/bench_c3_w16.json 2> $O/c3.err
timeout 600 python bench.py --steps 50 --warmup 5 --beads 1000 --cutoff 2.0 --replicas 16 --no-cpu-baseline --no-gpu-baseline > $O/bench_c5_coil1000.json 2> $O/c5a.err
timeout 600 python bench.py --steps 30 --warmup 5 --beads 2000 --cutoff 2.0 --replicas 16 --no-cpu-baseline --no-gpu-baseline > $O/bench_c5_coil2000.json 2> $O/c5b.err
timeout 600 python bench.py --steps 20 --warmup 3 --beads 5000 --cutoff 2.0 --replicas 16 --no-cpu-baseline --no-gpu-baseline > $O/bench_c5_coil5000.json 2> $O/c5c.err
timeout 600 python bench.py --steps 30 --warmup 5 --system globule --beads 1000 --cutoff 1.5 --replicas 16 --no-cpu-baseline --no-gpu-baseline > $O/bench_c5_glob1000.json 2> $O/c5d.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gpu-baseline --e2e-steps 1 --profile-steps 1 > /dev/null 2>&1
for f in $O/*.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), round(d['value'],1), d.get('e2e',{}).get('value'))"; done
tail -2 gpurun_out/pytest_configs_$TAG.log
