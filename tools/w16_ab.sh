cd $GRAFT_REPO_ROOT
for v in A B; do
  if [ $v = B ]; then export FCG_LIB_PATH=$PWD/paper_2602_13140_b200/libfcg_b.so; else unset FCG_LIB_PATH; fi
  timeout 300 python tools/diag_w16.py small_w16 coil269_w16 2>&1 | grep "err" | sed "s/^/$v /"
  timeout 300 python bench.py --config w16 --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['ms_per_step'], d['value'])"
done
