mkdir -p gpurun_out
PDGPU_K3_TM3=1 timeout 600 python -m pytest tests/test_gpu_scale.py -x -q -k "4096" > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
P="python profiles/pass_times.py 4096 4096 --reps 10 --batch 16"
for v in 0 1 0 1; do echo "tm3=$v $(PDGPU_K3_TM3=$v timeout 300 $P 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt; done
