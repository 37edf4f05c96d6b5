P="python profiles/pass_times.py 2048 2048 --batch 16 --reps 20"
for v in $AB_VARIANTS; do echo "== $v"; env $v $P 2>&1 | tail -1; env $v $P 2>&1 | tail -1; done
