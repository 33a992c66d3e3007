#!/bin/bash
# wgrad split-K clusters: kernel tests, lockstep parity of the small configs, per-op timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/cz
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv" > $O/kern.log 2>&1; echo kern rc=$?; tail -2 $O/kern.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cifar or resnet or lenet" > $O/par.log 2>&1; echo par rc=$?; tail -2 $O/par.log
python profiles/conv_bench.py --only cq. > $O/cb_cq.jsonl 2>&1
python profiles/conv_bench.py --only rn. >> $O/cb_cq.jsonl 2>&1
python profiles/conv_bench.py --only lenet. >> $O/cb_cq.jsonl 2>&1
cat $O/cb_cq.jsonl | cut -c1-120
for w in cifar10_quick resnet20 lenet; do timeout 300 python bench.py --workload $w --no-cpu-baseline > $O/b_$w.json 2>$O/b_$w.err; echo $w rc=$?; tail -1 $O/b_$w.json | cut -c1-260; done
