#!/bin/bash
# other BASELINE workloads + fc6 GEMM profile
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
for w in cifar10_quick lenet resnet20 pg_mlp; do
  python bench.py --workload $w --steps 30 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err
done
python bench.py --workload cifar10_quick --dtype f64 --steps 20 --warmup 5 > $O/bench_cifar10_quick_f64.json 2> $O/bench_cq64.err
python profiles/conv_bench.py --only fc6 --ops fwd,bwd --reps 1 > $O/plain_fc6.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|transpose|colsum" -s 2 -c 6 -o $O/fc6 -f \
    python profiles/conv_bench.py --only fc6 --ops fwd,bwd --reps 1 > $O/ncu_fc6.log 2>&1
echo prof done
