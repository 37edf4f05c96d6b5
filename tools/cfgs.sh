# secondary configs of the bench line (CG, sweep) under env variants
for v in $AB_VARIANTS; do echo "== $v"; env $v python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c '
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d["configs"]
print(d["ms_per_step"], {k:(round(v.get("solve_ms",0),2) if "solve_ms" in v else None) for k,v in c.items() if "cg" in k})
print({k:round(v["ms_per_step"],4) for k,v in c["config2_sweep_b16"].items()}, c["config5_vv"]["ms_per_step"], c["config4_matvec_256"]["ms_per_matvec"])
'; done
