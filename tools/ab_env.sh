# A/B of environment variants at 4096^2 x 16 (GPU box): AB_VARIANTS="A=1 B=2" bash tools/ab_env.sh
P="python profiles/pass_times.py 4096 4096 --batch 16 --reps 10"
nvidia-smi --query-gpu=name,serial,uuid --format=csv,noheader
for v in $AB_VARIANTS; do
  echo "== $v"
  env $v $P 2>&1 | tail -1
  env $v $P 2>&1 | tail -1
done
