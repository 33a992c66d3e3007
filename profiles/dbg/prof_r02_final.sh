#!/bin/bash
# Round-2 evidence: AlexNet conv2 backward (the bench line's dominant layer op) kernels
# and conv3 forward under ncu --set full; the DRAM bytes of every kernel of conv2's
# backward; the launch list of one AlexNet step.  (gpurun brings back <= 64 MiB.)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/plain_c2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/r02_ax_conv2_bwd_dram.csv \
    python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/ncu_c2d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"conv_tap|conv_wtap" -s 2 -c 2 -o $O/r02_ax_conv2_bwd -f \
    python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/ncu_c2.log 2>&1
python profiles/conv_bench.py --only alexnet.conv3 --ops fwd --reps 1 > $O/plain_c3f.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:conv_tap -s 1 -c 1 -o $O/r02_ax_conv3_fwd -f \
    python profiles/conv_bench.py --only alexnet.conv3 --ops fwd --reps 1 > $O/ncu_c3f.log 2>&1
python profiles/prof_step.py 2 alexnet > $O/ps2_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_ax_launches.csv \
    python profiles/prof_step.py 2 alexnet > $O/ps2_ncu.log 2>&1
du -sh $O/*
echo prof done
