#!/bin/bash
# ncu captures: K3 tmreg / land at batch 2; K1 CF=1 / CF=0 at batch 16 (memory metrics only)
mkdir -p gpurun_out
P="python profiles/pass_times.py 4096 4096 --reps 1"
for k3 in tmreg land; do
PDGPU_K3=$k3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spectral2d" -s 3 -c 1 -o gpurun_out/prof_k3_$k3 $P --batch 2 > gpurun_out/ncu_k3_$k3.log 2>&1
done
for cf in 1 0; do
PDGPU_K1_CF=$cf timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct --clock-control none -k regex:"k_rfft_rows" -s 3 -c 2 --csv $P --batch 16 > gpurun_out/ncu_k1_cf$cf.csv 2>&1
done
echo done
