#!/bin/bash
# fused LRN+pool backward fast path: launch bounds (256) vs (256, 2); the tests on the default build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "lrn" 2>&1 | tail -1
L=paper_1810_02272_b200/lib/libcudadnn.so
cp $L /tmp/orig.so
for v in lb1 lb2; do
  cp build/variants/libcudadnn_$v.so $L
  echo "== $v"; python profiles/lrnpool_bench.py --fused-only 2>&1 | grep bwd
done
cp /tmp/orig.so $L
