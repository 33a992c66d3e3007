#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/red
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv" > $O/kern.log 2>&1; echo kern rc=$?; tail -2 $O/kern.log
timeout 900 python -m pytest tests/test_gpu_checkpoint.py tests/test_gpu_bench_size.py -x -q > $O/ck.log 2>&1; echo ck rc=$?; tail -2 $O/ck.log
python profiles/conv_bench.py --ops wgrad > $O/cb.jsonl 2>&1; cut -c1-110 $O/cb.jsonl
timeout 300 python bench.py --no-cpu-baseline > $O/b_alexnet.json 2> $O/b_alexnet.err; tail -1 $O/b_alexnet.json | cut -c1-300
