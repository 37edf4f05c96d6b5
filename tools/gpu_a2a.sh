mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_transpose.py -q > gpurun_out/a2a_t.log 2>&1; echo rc=$? >> gpurun_out/a2a_t.log
timeout 600 python bench.py --shard transpose --steps 5 --warmup 3 > gpurun_out/a2a_b.json 2> gpurun_out/a2a_b.err
timeout 1200 python tools/transpose_proj.py 4096 16 1 2 4 8 > gpurun_out/a2a_proj.log 2>&1
