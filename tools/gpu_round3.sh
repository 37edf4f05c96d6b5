#!/bin/bash
# One GPU call (round 2, final state): tests, bench line, launch list, ncu full
# captures of K1 / K3 / K5 summarised on the box (the reports stay there).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,serial,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t.log
timeout 900 python bench.py > gpurun_out/b.json 2> gpurun_out/b.err
B="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
B2="python bench.py --batch 2 --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra"
timeout 300 $B2 > gpurun_out/plain2.log 2>&1 || exit 0
: > gpurun_out/ncu_full_b2.txt
for k in k_rfft_rows k_spectral2d k_irfft_rows; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 -o /tmp/prof_$k -f $B2 > gpurun_out/ncu_$k.log 2>&1
  python profiles/ncu_summary.py /tmp/prof_$k.ncu-rep >> gpurun_out/ncu_full_b2.txt 2>&1
  python profiles/ncu_lines.py /tmp/prof_$k.ncu-rep $k 30 > gpurun_out/ncu_lines_$k.txt 2>&1
  rm -f /tmp/prof_$k.ncu-rep
done
echo done
