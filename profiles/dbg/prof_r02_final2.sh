#!/bin/bash
# Round-2 closing evidence (one B200): AlexNet step launch list; DRAM bytes of the
# roofline op (conv2 backward); ncu --set full of conv3/4/5 weight gradients (tensor
# pipe; metrics only, gpurun returns <= 64 MiB), the fused LRN+pool pair, the persistent fc6 dW GEMM and the fused PG-MLP
# kernel.  Each ncu command runs only after the same command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/fin
mkdir -p $O
python profiles/prof_step.py 2 alexnet > $O/ps_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ax_launches.csv \
    python profiles/prof_step.py 2 alexnet > $O/ps_ncu.log 2>&1
python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/plain_c2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/ax_conv2_bwd_dram.csv \
    python profiles/conv_bench.py --only alexnet.conv2 --ops dgrad,wgrad --reps 1 > $O/ncu_c2d.log 2>&1
for L in conv3 conv4 conv5; do
  python profiles/conv_bench.py --only alexnet.$L --ops wgrad --reps 1 > $O/plain_$L.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,sm__issue_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:conv_wtap -s 1 -c 1 -o $O/ax_${L}_wgrad -f \
      python profiles/conv_bench.py --only alexnet.$L --ops wgrad --reps 1 > $O/ncu_$L.log 2>&1
done
python profiles/lrnpool_bench.py --only norm1 --fused-only --reps 1 > $O/plain_lp.log 2>&1 &&
ncu --set full --clock-control none -k regex:lrn_maxpool -s 2 -c 2 -o $O/lrnpool -f \
    python profiles/lrnpool_bench.py --only norm1 --fused-only --reps 1 > $O/ncu_lp.log 2>&1
python profiles/conv_bench.py --only fc6 --ops bwd --reps 1 > $O/plain_fc6.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,sm__issue_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm_persist -s 1 -c 1 -o $O/fc6_dw -f \
    python profiles/conv_bench.py --only fc6 --ops bwd --reps 1 > $O/ncu_fc6.log 2>&1
python bench.py --workload pg_mlp --steps 3 --warmup 3 --no-cpu-baseline > $O/plain_pg.log 2>&1 &&
ncu --set full --clock-control none -k regex:mlp_pg -s 2 -c 1 -o $O/pg_mlp -f \
    python bench.py --workload pg_mlp --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_pg.log 2>&1


# summaries on the box; only the small full captures travel back
python profiles/ncu_kernel_summary.py conv3.wgrad=$O/ax_conv3_wgrad.ncu-rep conv4.wgrad=$O/ax_conv4_wgrad.ncu-rep \
    conv5.wgrad=$O/ax_conv5_wgrad.ncu-rep fc6.dW=$O/fc6_dw.ncu-rep norm1+pool1=$O/lrnpool.ncu-rep \
    pg_mlp.step=$O/pg_mlp.ncu-rep > $O/r02_ncu_kernels_final.txt 2>&1
python profiles/summarize_launches.py $O/ax_launches.csv 88 > $O/r02_launches_alexnet_step_final.txt 2>&1
rm -f $O/ax_conv3_wgrad.ncu-rep $O/ax_conv4_wgrad.ncu-rep $O/ax_conv5_wgrad.ncu-rep $O/fc6_dw.ncu-rep
du -sh $O
echo prof done
