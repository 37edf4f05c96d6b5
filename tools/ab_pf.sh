#!/bin/bash
mkdir -p gpurun_out
P="python profiles/pass_times.py 4096 4096 --reps 10 --batch 16"
for k5 in 32 64 100 148 200; do
  echo "K5_PF=$k5 $(PDGPU_K5_PF=$k5 timeout 300 $P 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt
done
for k1 in 2 3; do
  echo "K1_PF=$k1 $(PDGPU_K1_PF=$k1 timeout 300 $P 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt
done
P2="python profiles/pass_times.py 2048 2048 --reps 10 --batch 16"
P3="python profiles/pass_times.py 256 256 256 --reps 10"
P4="python profiles/pass_times.py 1024 1024 --reps 10 --batch 16"
for k5 in 0 148; do for p in "$P2" "$P3" "$P4"; do
  echo "K5_PF=$k5 $(PDGPU_K5_PF=$k5 timeout 300 $p 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt
done; done
echo done
