#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/full
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 $O/gpu_tests.log
for w in alexnet cifar10_quick resnet20; do timeout 400 python bench.py --workload $w --no-cpu-baseline > $O/b_$w.json 2>$O/b_$w.err; echo $w rc=$?; tail -1 $O/b_$w.json | cut -c1-200; done
