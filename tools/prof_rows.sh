# ncu full capture (source-level) of the 2D K1 / K3 / K5 at 4096^2, batch 2
B2="python bench.py --batch 2 --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra"
timeout 300 $B2 > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rfft_rows|k_spectral2d|k_irfft_rows" -s 3 -c 3 -o gpurun_out/prof_rows -f $B2 > gpurun_out/ncu_rows.log 2>&1
tail -2 gpurun_out/ncu_rows.log | cut -c1-300
