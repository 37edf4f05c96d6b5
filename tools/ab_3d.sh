#!/bin/bash
mkdir -p gpurun_out
for g in 0 148 296 592 1184; do echo "GPF=$g $(PDGPU_K5_GPF=$g timeout 300 python profiles/pass_times.py 256 256 256 --reps 10 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt; done
for g in 0 592; do echo "GPF=$g $(PDGPU_K5_GPF=$g timeout 300 python profiles/pass_times.py 512 512 --batch 16 --reps 10 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt; done
for g in 0 592; do echo "GPF=$g $(PDGPU_K5_GPF=$g timeout 300 python profiles/pass_times.py 128 128 128 --reps 10 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt; done
echo done
