#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_matvec.py tests/test_gpu_embedding.py -x -q > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
P="python profiles/pass_times.py 4096 4096 --reps 10"
for b in 16 2; do for k3 in tmreg split; do
  echo "K3=$k3 $(PDGPU_K3=$k3 timeout 300 $P --batch $b 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spectral2d" -s 3 -c 1 -o gpurun_out/prof_k3_tmreg python profiles/pass_times.py 4096 4096 --reps 1 --batch 2 > gpurun_out/ncu_k3.log 2>&1
echo done
