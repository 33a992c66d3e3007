#!/bin/bash
# Round-2 evidence: AlexNet conv2 backward (the bench line's dominant layer op) and the
# other dominant kernels under ncu --set full; the launch list of one AlexNet step.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/plain_c2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -o $O/r02_ax_conv2_bwd -f \
    python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/ncu_c2.log 2>&1
python profiles/conv_bench.py --only alexnet.conv3 --ops fwd --reps 1 > $O/plain_c3f.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:conv_tap -s 1 -c 1 -o $O/r02_ax_conv3_fwd -f \
    python profiles/conv_bench.py --only alexnet.conv3 --ops fwd --reps 1 > $O/ncu_c3f.log 2>&1
python profiles/prof_step.py 2 alexnet > $O/ps2_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_ax_launches.csv \
    python profiles/prof_step.py 2 alexnet > $O/ps2_ncu.log 2>&1
echo prof done
