#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bench_size.py -x -q -k "gemm or ip or conv or bench" 2>&1 | tail -2
python profiles/conv_bench.py --only fc --reps 20 2>&1 | cut -c1-90
python profiles/conv_bench.py --only cq.ip --reps 20 2>&1 | cut -c1-90
