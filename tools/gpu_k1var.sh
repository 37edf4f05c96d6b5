B="python bench.py --no-cpu --no-e2e --no-extra"
for v in "PDGPU_NO_K1_PIPE=1 PDGPU_K1_ROWS=2" "PDGPU_NO_K1_PIPE=1 PDGPU_K1_ROWS=1" "PDGPU_K1_ROWS=1" "PDGPU_K5_ROWS=2" "PDGPU_K5_ROWS=4"; do
  echo "$v $(env PDGPU_K1_CL=1 $v $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["passes_ms_per_step"])')" >> gpurun_out/k1var.txt
done
