mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scale.py tests/test_gpu_matvec.py tests/test_gpu_wrap_faces.py -x -q > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
for d in "256 256 256" "128 128 128"; do timeout 300 python profiles/pass_times.py $d --reps 10 2>&1 | tail -1 >> gpurun_out/ab_passes.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spectral<|k_cfft" -s 3 -c 3 -o gpurun_out/prof_3dk3 python profiles/pass_times.py 256 256 256 --reps 1 > gpurun_out/ncu_3dk3.log 2>&1
