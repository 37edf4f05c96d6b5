mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
for v in 1 0; do echo "pdl=$v" >> gpurun_out/ab_passes.txt; PDGPU_PDL=$v timeout 300 python tools/cg_iter.py >> gpurun_out/ab_passes.txt 2>&1; done
