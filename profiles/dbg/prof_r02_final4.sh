#!/bin/bash
# Round-2 closing evidence at the final build (one B200), second closing pass:
#  1. bench lines of every workload + the reference arms (profiles/dbg/bench_all.sh)
#  2. launch list of the default bench command itself (AlexNet b256, graph replay)
#  3. launch list (time + DRAM bytes) of one eager AlexNet step (profiles/prof_step.py)
#  4. DRAM bytes of the roofline op (conv2 backward: dgrad + wgrad kernels)
#  5. ncu --set full metrics of conv2's backward kernels and conv1 forward (summaries only)
# Each ncu command runs only after the same command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/fin6
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
bash profiles/dbg/bench_all.sh $O/bench
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_small.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_ncu.log 2>&1
python profiles/prof_step.py 2 alexnet > $O/ps_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/ax_step_launches.csv python profiles/prof_step.py 2 alexnet > $O/ps_ncu.log 2>&1
python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/plain_c2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/ax_conv2_bwd_dram.csv python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/ncu_c2d.log 2>&1
ncu --set full --clock-control none -k regex:"conv_tap|conv_wtap" -s 3 -c 3 -o $O/c2 -f \
    python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/ncu_c2.log 2>&1
python profiles/conv_bench.py --only alexnet.conv1 --ops fwd --reps 1 > $O/plain_c1.log 2>&1 &&
ncu --set full --clock-control none -k regex:"conv_tap" -s 1 -c 1 -o $O/c1 -f \
    python profiles/conv_bench.py --only alexnet.conv1 --ops fwd --reps 1 > $O/ncu_c1.log 2>&1
python profiles/ncu_kernel_summary.py conv2.bwd=$O/c2.ncu-rep conv1.fwd=$O/c1.ncu-rep > $O/r02_ncu_kernels_closing.txt 2>&1
for r in c2 c1; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null; done
rm -f $O/*.ncu-rep
python profiles/summarize_launches.py $O/ax_step_launches.csv 88 > $O/r02_launches_alexnet_step_closing.txt 2>&1
python profiles/summarize_launches.py $O/bench_launches.csv > $O/r02_launches_bench_alexnet.txt 2>&1
du -sh $O
echo prof done
# 6. ResNet-20 step launch list (time + DRAM bytes) and the fused LRN+pool / pooling benches
python profiles/prof_step.py 2 resnet20 > $O/rn_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/rn_step_launches.csv python profiles/prof_step.py 2 resnet20 > $O/rn_ncu.log 2>&1
timeout 300 python profiles/lrnpool_bench.py > $O/lrnpool.jsonl 2>&1
timeout 300 python profiles/pool_bench.py > $O/pool.jsonl 2>&1
