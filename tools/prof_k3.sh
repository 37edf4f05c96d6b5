# ncu full capture (source-level) of the 2D K3 at 4096^2, batch 2
B2="python bench.py --batch 2 --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra"
timeout 300 $B2 > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spectral2d" -s 1 -c 1 -o gpurun_out/prof_k3 -f $B2 > gpurun_out/ncu_k3.log 2>&1
python profiles/pass_times.py 4096 4096 --batch 16 --reps 10 | tail -1
