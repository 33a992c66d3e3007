#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/pool
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "pool" > $O/kern.log 2>&1; echo kern rc=$?; tail -2 $O/kern.log
python profiles/pool_bench.py > $O/pool_bench.jsonl 2> $O/pool_bench.err; cut -c1-130 $O/pool_bench.jsonl | head -6
python profiles/pool_bench.py --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__issue_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:max_pool -c 4 --csv --log-file $O/ncu_pool.csv python profiles/pool_bench.py --reps 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader([l for l in open('gpurun_out/pool/ncu_pool.csv') if l.startswith('"')])]
for r in rows: print(r['ID'], r['Kernel Name'][:40], r['Metric Name'], r['Metric Value'])
PY
