#!/bin/bash
# Headline + secondary BASELINE configs through bench.py (one GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "$tag exit $?"; }
run c2_fp32 --steps 200 --warmup 20
run c3_w16 --config w16 --steps 200 --warmup 20 --no-cpu-baseline
run c5_coil1000 --system coil --beads 1000 --cutoff 2.0 --replicas 16 --steps 50 --warmup 5 --no-cpu-baseline
run c5_coil2000 --system coil --beads 2000 --cutoff 2.0 --replicas 16 --steps 30 --warmup 3 --no-cpu-baseline
run c5_coil5000 --system coil --beads 5000 --cutoff 2.0 --replicas 16 --steps 10 --warmup 3 --no-cpu-baseline
run c5_glob1000 --system globule --beads 1000 --cutoff 1.5 --replicas 16 --steps 30 --warmup 3 --no-cpu-baseline
run ref_c1 --impl reference --steps 3 --warmup 1
