#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/abcz
mkdir -p $O
export CDNN_DBG_CZ_T=1
for v in 2 4 8 off; do
  if [ $v = off ]; then export CDNN_DBG_CZ_OFF=1; else export CDNN_DBG_CZ=$v; fi
  echo "== $v"
  CDNN_DBG_CZ_PRINT=1 python profiles/conv_bench.py --only cq.conv2 --ops wgrad --reps 1 2>&1 | grep wtap | sort -u
  CDNN_DBG_CZ_PRINT=1 python profiles/conv_bench.py --only rn.stage1 --ops wgrad --reps 1 2>&1 | grep wtap | sort -u
  python profiles/conv_bench.py --only cq.conv --ops wgrad > $O/cb_$v.jsonl 2>&1
  python profiles/conv_bench.py --only rn. --ops wgrad >> $O/cb_$v.jsonl 2>&1
  python profiles/conv_bench.py --only lenet. --ops wgrad >> $O/cb_$v.jsonl 2>&1
  cat $O/cb_$v.jsonl | cut -c1-100
done
