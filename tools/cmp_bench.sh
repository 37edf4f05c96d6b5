mkdir -p gpurun_out
P="python profiles/pass_times.py 4096 4096 --reps 10 --batch 16"
echo "pt1 $($P 2>&1 | tail -1)" > gpurun_out/cmp.txt
python bench.py --no-cpu --no-e2e --no-extra > gpurun_out/cmp_b.json 2>/dev/null
echo "pt2 $($P 2>&1 | tail -1)" >> gpurun_out/cmp.txt
PDGPU_K5_PF=0 python bench.py --no-cpu --no-e2e --no-extra > gpurun_out/cmp_b0.json 2>/dev/null
echo "pt3 $(PDGPU_K5_PF=0 $P 2>&1 | tail -1)" >> gpurun_out/cmp.txt
