# Caffe-ordered wgrad split reduce vs the (m, n)-tiled one (temporary CDNN_TMP_OLD_REDUCE)
mkdir -p gpurun_out/rd
for rep in 1 2; do
  timeout 300 python profiles/conv_bench.py --only alexnet --ops wgrad --reps 20 > gpurun_out/rd/new_$rep.jsonl 2>&1
  CDNN_TMP_OLD_REDUCE=1 timeout 300 python profiles/conv_bench.py --only alexnet --ops wgrad --reps 20 > gpurun_out/rd/old_$rep.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bench_size.py -x -q -k "conv or alexnet" > gpurun_out/rd/tests.log 2>&1
python profiles/prof_step.py 2 alexnet > gpurun_out/rd/ps.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rd/launches.csv python profiles/prof_step.py 2 alexnet > /dev/null 2>&1
