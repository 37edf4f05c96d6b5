python -m pytest tests -m gpu -x -q > gpurun_out/t2.log 2>&1
python bench.py > gpurun_out/b2.json 2> gpurun_out/b2.err
B="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
B2="python bench.py --batch 2 --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra"
$B2 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_rfft_rows|k_spectral2d_duo|k_irfft_rows|k_wrap" -s 4 -c 4 -o gpurun_out/prof $B2 > gpurun_out/ncu2.log 2>&1
echo done
