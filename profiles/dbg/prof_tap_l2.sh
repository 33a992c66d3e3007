# L2 / tensor-pipe profile of the 13x13 tap convolutions (AlexNet conv4 forward, conv5
# backward-data) and the AlexNet bench after the LRN+pool forward prefetch ring.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/l2
mkdir -p $O
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python profiles/conv_bench.py --only alexnet.conv5 --ops dgrad --reps 3 > $O/c5.log 2>&1 &&
ncu --set full --clock-control none -k regex:"conv_tap" -s 1 -c 1 -o $O/c5d -f \
    python profiles/conv_bench.py --only alexnet.conv5 --ops dgrad --reps 1 > $O/ncu_c5.log 2>&1
python profiles/conv_bench.py --only alexnet.conv4 --ops fwd --reps 3 > $O/c4.log 2>&1 &&
ncu --set full --clock-control none -k regex:"conv_tap" -s 1 -c 1 -o $O/c4f -f \
    python profiles/conv_bench.py --only alexnet.conv4 --ops fwd --reps 1 > $O/ncu_c4.log 2>&1
for r in c5d c4f; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null; done
rm -f $O/*.ncu-rep
