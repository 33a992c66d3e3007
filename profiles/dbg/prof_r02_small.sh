#!/bin/bash
# Launch lists of one CIFAR-quick / ResNet-20 step (the small-channel path), and the
# current pooling / fused LRN+pool kernel bandwidths.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/small
mkdir -p $O
for w in cifar10_quick resnet20; do
  python profiles/prof_step.py 2 $w > $O/ps_$w.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${w}_launches.csv \
      python profiles/prof_step.py 2 $w > $O/ps_ncu_$w.log 2>&1
done
python profiles/pool_bench.py > $O/pool_bench.jsonl 2> $O/pool_bench.err
python profiles/lrnpool_bench.py > $O/lrnpool_bench.jsonl 2> $O/lrnpool_bench.err
echo done
