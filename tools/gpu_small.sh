#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t.log
timeout 300 python tools/cg_iter.py > gpurun_out/cg_iter.log 2>&1
for v in 0 1; do
  if [ $v = 1 ]; then export PDGPU_WRAP_GENERIC=1; fi
  echo "generic=$v" >> gpurun_out/passes.txt
  for d in "128 128 128" "256 256 256" "1024 1024" "128 128"; do timeout 300 python profiles/pass_times.py $d --reps 10 2>&1 | tail -1 >> gpurun_out/passes.txt; done
  timeout 300 python profiles/pass_times.py 4096 4096 --batch 16 --reps 10 2>&1 | tail -1 >> gpurun_out/passes.txt
done
unset PDGPU_WRAP_GENERIC
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cg1_launches.csv python tools/small_prof.py 128 3 > /dev/null 2>&1
echo done
