#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/poolp
mkdir -p $O
python profiles/pool_bench.py --reps 1 > $O/plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:"max_pool_fwd_k2|max_pool_bwd_blk" -c 2 -o $O/pp -f \
  python profiles/pool_bench.py --reps 1 > $O/ncu.log 2>&1
ncu -i $O/pp.ncu-rep --page raw --csv > $O/pp_raw.csv 2>/dev/null
ncu -i $O/pp.ncu-rep --page source --csv --print-source sass > $O/pp_sass.csv 2>/dev/null
rm -f $O/pp.ncu-rep
