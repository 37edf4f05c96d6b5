python -m pytest tests -m gpu -x -q > gpurun_out/t9.log 2>&1
B="python bench.py --no-cpu --no-e2e --no-extra"
for v in "PDGPU_X=0" "PDGPU_NO_K1_DUO=1"; do
  echo "$v $(env $v $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["passes_ms_per_step"])')" >> gpurun_out/k1duo.txt
done
