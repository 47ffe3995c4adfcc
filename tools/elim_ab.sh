cd $GRAFT_REPO_ROOT
for v in A B A B; do
  if [ $v = B ]; then export FCG_LIB_PATH=$PWD/paper_2602_13140_b200/libfcg_b.so; else unset FCG_LIB_PATH; fi
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-gpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['ms_per_step'])"
done
