mkdir -p gpurun_out/sw
for cfg in "40 224 512 1" "40 224 1024 1" "24 224 1024 1" "64 224 1024 1" "40 110 512 2" "24 110 512 2" "16 72 256 3" "12 56 256 4"; do
  set -- $cfg
  echo "== target=$1 smem=$2 threads=$3 per_sm=$4" >> gpurun_out/sw/sweep.txt
  CDNN_STAGE_TARGET_KB=$1 CDNN_STAGE_SMEM_KB=$2 CDNN_STAGE_THREADS=$3 CDNN_STAGE_PER_SM=$4 timeout 120 python profiles/pool_bench.py --reps 10 2>&1 | grep -E "alexnet|cq.pool1|Error|error" >> gpurun_out/sw/sweep.txt
done
