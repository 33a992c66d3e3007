# LRN+pool forward: cp.async prefetch depth sweep (temporary CDNN_TMP_PF switch)
mkdir -p gpurun_out/pf
for pf in 2 3 4; do
  echo "== PF=$pf" >> gpurun_out/pf/sweep.txt
  CDNN_TMP_PF=$pf timeout 120 python profiles/lrnpool_bench.py --fused-only 2>&1 | grep fwd >> gpurun_out/pf/sweep.txt
done
CDNN_TMP_PF=2 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "lrn_pool" > gpurun_out/pf/t8.log 2>&1
CDNN_TMP_PF=3 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "lrn_pool" > gpurun_out/pf/t6.log 2>&1
