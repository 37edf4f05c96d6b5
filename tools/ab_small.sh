#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab_t.log 2>&1; echo "rc=$?" >> gpurun_out/ab_t.log
timeout 300 python tools/cg_iter.py > gpurun_out/ab_passes.txt 2>&1
for d in "128 128" "1024 1024" "128 128 128"; do timeout 300 python profiles/pass_times.py $d --reps 10 2>&1 | tail -1 >> gpurun_out/ab_passes.txt; done
timeout 300 python profiles/pass_times.py 4096 4096 --batch 16 --reps 10 2>&1 | tail -1 >> gpurun_out/ab_passes.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cg1_launches.csv python tools/small_prof.py 128 3 > /dev/null 2>&1
echo done
