mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
