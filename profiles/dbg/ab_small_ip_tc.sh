# A/B: small InnerProducts (LeNet / CIFAR-quick, <= 2^26 MACs) on the exact-fp32 SIMT engines
# (default) vs forced onto the tcgen05 3xTF32 GEMM (temporary CDNN_AB_FORCE_TC switch).
mkdir -p gpurun_out/ab
for wl in lenet cifar10_quick; do
  for rep in 1 2; do
    timeout 300 python bench.py --workload $wl --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab/${wl}_simt_$rep.json
    CDNN_AB_FORCE_TC=1 timeout 300 python bench.py --workload $wl --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab/${wl}_tc_$rep.json
  done
  CDNN_AB_FORCE_TC=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "$wl" > gpurun_out/ab/${wl}_tc_parity.log 2>&1
  for mode in simt tc; do
    env_=""; [ $mode = tc ] && env_="CDNN_AB_FORCE_TC=1"
    env $env_ timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab/${wl}_${mode}_launches.csv python profiles/prof_step.py 2 $wl > /dev/null 2>&1
  done
done
