#!/bin/bash
# Round-2 bench lines for every workload (one B200): product arm and the reference arm.
out=${1:-gpurun_out/bench_all}
mkdir -p $out
for w in alexnet cifar10_quick lenet resnet20 pg_mlp; do
  timeout 400 python bench.py --workload $w > $out/$w.json 2> $out/$w.err
  echo "$w rc=$? $(tail -1 $out/$w.json | cut -c1-200)"
done
timeout 400 python bench.py --workload cifar10_quick --dtype f64 > $out/cifar10_quick_f64.json 2> $out/cifar10_quick_f64.err
echo "cq f64 rc=$? $(tail -1 $out/cifar10_quick_f64.json | cut -c1-200)"
for w in alexnet pg_mlp; do
  timeout 600 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > $out/ref_$w.json 2> $out/ref_$w.err
  echo "ref $w rc=$? $(tail -1 $out/ref_$w.json | cut -c1-200)"
done
