#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "$1" > $O/it_tests.log 2>&1; echo "tests exit $?" >> $O/it_tests.log
timeout 300 python bench.py --no-cpu-baseline > $O/it_cq.json 2> $O/it_cq.err
timeout 300 python bench.py --no-cpu-baseline --workload alexnet > $O/it_ax.json 2> $O/it_ax.err
