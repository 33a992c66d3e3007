#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/lrnf
mkdir -p $O
python profiles/lrnpool_bench.py --only norm1 --fused-only --reps 1 > $O/plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:lrn_maxpool_fwd -c 1 -o $O/lb -f \
  python profiles/lrnpool_bench.py --only norm1 --fused-only --reps 1 > $O/ncu.log 2>&1
ncu -i $O/lb.ncu-rep --page raw --csv > $O/lb_raw.csv 2>/dev/null
ncu -i $O/lb.ncu-rep --page source --csv --print-source sass > $O/lb_sass.csv 2>/dev/null
rm -f $O/lb.ncu-rep
ls -la $O
