B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-extra"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], {k:round(v,3) for k,v in d["roofline"]["passes_ms_per_step"].items()})'
for v in ${AB_VARIANTS:-""}; do echo "$v"; env $v $B 2>/dev/null | python -c "$P"; done
