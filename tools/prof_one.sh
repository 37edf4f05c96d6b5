# ncu full capture (source-level) of one 2D pass at 4096^2, batch 2: bash tools/prof_one.sh REGEX NAME
B2="python bench.py --batch 2 --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra"
timeout 300 $B2 > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s 1 -c 1 -o gpurun_out/$2 -f $B2 > gpurun_out/ncu_$2.log 2>&1
tail -1 gpurun_out/ncu_$2.log | cut -c1-200
