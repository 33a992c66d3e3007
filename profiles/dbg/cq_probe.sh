#!/bin/bash
# CIFAR-quick conv kernel probe: timings per route, tap traces, one ncu --set full per kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
python profiles/conv_bench.py --only cq. > $O/cq_default.txt 2>&1
CDNN_CONV_TMA=0 python profiles/conv_bench.py --only cq. > $O/cq_notma.txt 2>&1
CDNN_CONV_TMA=0 CDNN_TAP_TRACE=1 python profiles/conv_bench.py --only cq.conv1 --reps 2 > $O/cq_trace1.txt 2>&1
CDNN_TAP_TRACE=1 python profiles/conv_bench.py --only cq.conv2 --reps 2 > $O/cq_trace2.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tap -c 1 -o $O/cq_conv2_tap -f python profiles/conv_bench.py --only cq.conv2 --reps 1 > $O/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tma -c 1 -o $O/cq_conv1_tma -f python profiles/conv_bench.py --only cq.conv1 --reps 1 > $O/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_wtap -c 1 -o $O/cq_conv2_wtap -f python profiles/conv_bench.py --only cq.conv2 --reps 1 > $O/ncu3.log 2>&1
