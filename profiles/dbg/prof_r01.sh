#!/bin/bash
# Round-1 ncu evidence: CIFAR-quick step launch list with DRAM bytes, the headline's dominant
# kernels, and AlexNet tensor-core / HBM kernels (one GPU process per ncu run).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
ncu --metrics $M --csv python profiles/prof_step.py 2 > $O/cq_dram.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/prof_step.py 2 > $O/cq_launches.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tap -s 3 -c 1 -o $O/cq_conv2_dgrad -f python profiles/conv_bench.py --only cq.conv2 --reps 1 > $O/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tap -c 1 -o $O/ax_conv3_fwd -f python profiles/conv_bench.py --only alexnet.conv3 --reps 1 > $O/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o $O/ax_fc6_fwd -f python profiles/conv_bench.py --only fc6 --reps 1 > $O/ncu_c.log 2>&1
ncu --set full --clock-control none -k regex:"sgd|relu_bwd|max_pool_fwd" -c 3 -o $O/ax_elem -f python profiles/prof_step.py 1 alexnet > $O/ncu_d.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/prof_step.py 1 alexnet > $O/ax_launches.csv 2>&1
