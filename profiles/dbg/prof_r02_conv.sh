#!/bin/bash
# Round-2 ncu evidence for the AlexNet convolution kernels (one GPU process per ncu run;
# each command ran plain first).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
python profiles/conv_bench.py --only alexnet --reps 10 > $O/conv_bench_ax.jsonl 2>&1 || exit 1
python profiles/conv_bench.py --only alexnet --reps 10 --math tf32 > $O/conv_bench_ax_tf32.jsonl 2>&1 || exit 1
python profiles/conv_bench.py --only alexnet.conv3 --ops wgrad,fwd --reps 1 > $O/plain3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"conv_wtap|conv_tap" -s 1 -c 2 -o $O/ax_conv3 -f \
    python profiles/conv_bench.py --only alexnet.conv3 --ops wgrad,fwd --reps 1 > $O/ncu_conv3.log 2>&1
python profiles/conv_bench.py --only alexnet.conv2 --ops wgrad --reps 1 > $O/plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"conv_wtap" -s 1 -c 1 -o $O/ax_conv2_wgrad -f \
    python profiles/conv_bench.py --only alexnet.conv2 --ops wgrad --reps 1 > $O/ncu_conv2.log 2>&1
echo prof done
