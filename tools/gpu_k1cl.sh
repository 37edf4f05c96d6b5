python -m pytest tests/test_gpu_embedding.py tests/test_gpu_matvec.py -m gpu -x -q > gpurun_out/t4.log 2>&1
B="python bench.py --no-cpu --no-e2e --no-extra"
for v in "4 2" "8 1" "2 2" "2 1" "4 1"; do
  set -- $v
  echo "CL=$1 TR=$2 $(PDGPU_K1_CL=$1 PDGPU_K1_CLTR=$2 $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["passes_ms_per_step"]["K1_rfft_x"])')" >> gpurun_out/k1cl2.txt
done
