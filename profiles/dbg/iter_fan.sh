#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/fan
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "fan or scale or eltwise" > $O/kern.log 2>&1; echo kern rc=$?; tail -2 $O/kern.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp_product.py -x -q -k "resnet" > $O/par.log 2>&1; echo par rc=$?; tail -2 $O/par.log
for w in resnet20 alexnet; do timeout 300 python bench.py --workload $w --no-cpu-baseline > $O/b_$w.json 2>$O/b_$w.err; echo $w rc=$?; tail -1 $O/b_$w.json | cut -c1-250; done
