#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_scale.py tests/test_gpu_embedding.py tests/test_gpu_golden.py -x -q > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
for v in 0 1; do
 if [ $v = 1 ]; then export PDGPU_WRAP_NOFACE=1; fi
 for d in "256 256 256" "128 128 128"; do echo "noface=$v $(timeout 300 python profiles/pass_times.py $d --reps 10 2>&1 | tail -1)" >> gpurun_out/ab_passes.txt; done
done
unset PDGPU_WRAP_NOFACE
timeout 300 python tools/cg_iter.py >> gpurun_out/ab_passes.txt 2>&1
echo done
