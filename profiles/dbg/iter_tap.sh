#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/tap
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv" > $O/kern.log 2>&1; echo kern rc=$?; tail -2 $O/kern.log
python profiles/conv_bench.py --ops fwd,dgrad,dgrad_gate > $O/cb.jsonl 2>&1; cut -c1-110 $O/cb.jsonl
