#!/bin/bash
# conv1 forward / weight gradient (space-to-depth, 48 channels): ncu --set full of the
# tap kernels, with source to read stall reasons.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/c1
mkdir -p $O
python profiles/conv_bench.py --only alexnet.conv1 --ops fwd,wgrad --reps 1 > $O/plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"conv_tap|conv_wtap" -c 2 -o $O/c1 -f \
  python profiles/conv_bench.py --only alexnet.conv1 --ops fwd,wgrad --reps 1 > $O/ncu.log 2>&1
python profiles/conv_bench.py --only alexnet.conv3 --ops fwd --reps 1 > $O/plain3.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"conv_tap" -c 1 -o $O/c3 -f \
  python profiles/conv_bench.py --only alexnet.conv3 --ops fwd --reps 1 > $O/ncu3.log 2>&1
python profiles/ncu_kernel_summary.py conv1=$O/c1.ncu-rep conv3.fwd=$O/c3.ncu-rep
ls -la $O
for r in c1 c3; do
  ncu -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
