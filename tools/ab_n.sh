# AB_N=1024 AB_VARIANTS="A=1 B=2" bash tools/ab_n.sh
P="python profiles/pass_times.py $AB_N $AB_N --batch 16 --reps 20"
for v in $AB_VARIANTS; do echo "== $v"; env $v $P 2>&1 | tail -1; env $v $P 2>&1 | tail -1; done
