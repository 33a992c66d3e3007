#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in 0 1; do
  echo "== nbuf1=$v"
  if [ $v = 1 ]; then export CDNN_DBG_NBUF1=1; fi
  python profiles/conv_bench.py --only alexnet.conv --ops fwd,dgrad 2>&1 | grep -E '"op"' | cut -c1-75
done
