python -m pytest tests -m gpu -x -q > gpurun_out/t23.log 2>&1
python tools/cg_iter.py > gpurun_out/cgiter2.txt 2>&1
PDGPU_CG_HOSTLOOP=1 python tools/cg_iter.py >> gpurun_out/cgiter2.txt 2>&1
for a in "128 128 128" "256 256 256" "4096 4096 --batch 16"; do python profiles/pass_times.py $a >> gpurun_out/cgiter2.txt 2>&1; done
