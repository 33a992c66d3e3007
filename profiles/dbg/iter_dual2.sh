#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bench_size.py -x -q -k "conv or bench or ip" 2>&1 | tail -1
for i in 1 2; do python profiles/conv_bench.py --only alexnet.conv --ops fwd,dgrad 2>&1 | grep -E '"op"' | cut -c1-75; done
for i in 1 2 3; do REPS=5 timeout 60 python profiles/dbg/ipbwd_probe.py 256 4096 4096 both 2>&1 | tail -1; done
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/b_ax.json 2>&1; tail -1 gpurun_out/b_ax.json | cut -c1-200
