#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv" 2>&1 | tail -1
CDNN_DBG_TPSP=1 python profiles/conv_bench.py --only alexnet.conv --ops fwd,dgrad --reps 1 2>&1 | grep '^tap' | sort -u
for v in "TPS=1" "TPSD=4" "TPSD=6" "TPS=2" "TPS=3" "TPS=4"; do
  echo "== $v"
  env CDNN_DBG_$v python profiles/conv_bench.py --only alexnet.conv --ops fwd,dgrad 2>&1 | grep -E '"op"' | cut -c1-75
done
for v in "TPS=1" "TPSD=4"; do
  echo "== small $v"
  env CDNN_DBG_$v python profiles/conv_bench.py --ops fwd,dgrad 2>&1 | grep -E '"op": "(cq|rn|lenet)' | cut -c1-75
done
