#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or ip" 2>&1 | tail -1
for i in 1 2 3; do REPS=5 timeout 60 python profiles/dbg/ipbwd_probe.py 256 4096 4096 both 2>&1 | tail -1; done
REPS=5 timeout 60 python profiles/dbg/ipbwd_probe.py 256 9216 4096 both 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_bench_size.py -x -q 2>&1 | tail -1
python profiles/conv_bench.py --only fc --reps 20 2>&1 | cut -c1-90
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/b_ax2.json 2>&1; tail -1 gpurun_out/b_ax2.json | cut -c1-200
