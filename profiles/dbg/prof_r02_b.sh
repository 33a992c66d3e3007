#!/bin/bash
# conv wgrad after the load-before-wait staging change; LRN+pool fused kernels (ncu)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
python profiles/conv_bench.py --only alexnet --ops wgrad --reps 10 > $O/conv_wgrad_b.jsonl 2>&1
python profiles/conv_bench.py --only alexnet --ops wgrad --reps 10 --math tf32 >> $O/conv_wgrad_b.jsonl 2>&1
python profiles/lrnpool_bench.py > $O/lrnpool_bench.jsonl 2>&1
python profiles/lrnpool_bench.py --only norm1 --fused-only --reps 1 > $O/plain_lp.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"lrn_maxpool" -s 2 -c 2 -o $O/lrnpool -f \
    python profiles/lrnpool_bench.py --only norm1 --fused-only --reps 1 > $O/ncu_lp.log 2>&1
python profiles/conv_bench.py --only alexnet.conv3 --ops wgrad --reps 1 > $O/plain3b.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"conv_wtap" -s 1 -c 1 -o $O/ax_conv3_wgrad_b -f \
    python profiles/conv_bench.py --only alexnet.conv3 --ops wgrad --reps 1 > $O/ncu_conv3b.log 2>&1
echo prof done
