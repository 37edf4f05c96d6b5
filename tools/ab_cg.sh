mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scale.py tests/test_gpu_golden.py tests/test_gpu_embedding.py -x -q > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
for g in 148 296 592; do echo "grid=$g" >> gpurun_out/ab_passes.txt; PDGPU_CG_GRID=$g timeout 300 python tools/cg_iter.py >> gpurun_out/ab_passes.txt 2>&1; done
