#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/lrn
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "lrn" > $O/kern.log 2>&1; echo kern rc=$?; tail -2 $O/kern.log
python profiles/lrnpool_bench.py > $O/lrnpool_bench.jsonl 2> $O/lrnpool_bench.err; cat $O/lrnpool_bench.jsonl
