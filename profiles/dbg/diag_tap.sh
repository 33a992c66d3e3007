#!/bin/bash
# Bottleneck diagnosis of the tap kernel (temporary build): 1 = weights TMA'd once per tile,
# 2 = no input staging, 4 = no epilogue stores, 8 = one k8 step of MMAs per tap
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for d in 0 1 2 4 8 3 9 10; do
  echo "== diag $d"
  CDNN_TAP_DIAG=$d python profiles/conv_bench.py --only alexnet.conv --ops fwd,dgrad 2>&1 | grep -E 'conv(1|2|3)\.(fwd|dgrad)"' | cut -c1-90
done
