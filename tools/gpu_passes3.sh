python -m pytest tests -m gpu -x -q > gpurun_out/t29.log 2>&1
for a in "128 128 128" "256 256 256" "512 512 --batch 16" "1024 1024 --batch 16"; do python profiles/pass_times.py $a >> gpurun_out/p29.txt 2>&1; PDGPU_K5_TMA=0 python profiles/pass_times.py $a >> gpurun_out/p29.txt 2>&1; done
