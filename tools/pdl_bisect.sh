cd $GRAFT_REPO_ROOT
T="tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k small0"
for v in v1 v2 default; do
  L=$PWD/paper_2602_13140_b200/libfcg_$v.so; [ $v = default ] && L=$PWD/paper_2602_13140_b200/libfcg.so
  for r in 1 2 3; do
    res=$(FCG_PDL=0x20 FCG_LIB_PATH=$L timeout 300 python -m pytest $T 2>&1 | tail -1)
    echo "$v run$r: $res"
  done
done
