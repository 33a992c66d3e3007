# LRN+pool backward with the cp.async gather ring: 3 vs 2 blocks per SM (temporary CDNN_TMP_MB2)
mkdir -p gpurun_out/lb
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "lrn" > gpurun_out/lb/t3.log 2>&1
CDNN_TMP_MB2=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "lrn_pool" > gpurun_out/lb/t2.log 2>&1
timeout 120 python profiles/lrnpool_bench.py --fused-only > gpurun_out/lb/mb3.jsonl 2>&1
CDNN_TMP_MB2=1 timeout 120 python profiles/lrnpool_bench.py --fused-only > gpurun_out/lb/mb2.jsonl 2>&1
