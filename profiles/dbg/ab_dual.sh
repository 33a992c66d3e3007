#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv" 2>&1 | tail -2
for v in 0 1; do
  echo "== nodual=$v"
  if [ $v = 1 ]; then export CDNN_DBG_NODUAL=1; fi
  timeout 300 python profiles/conv_bench.py --ops fwd,dgrad 2>&1 | grep -E '"op": "(alexnet|cq|rn)\.conv|rn\.' | cut -c1-75
done
