python -m pytest tests -m gpu -x -q > gpurun_out/t11.log 2>&1
for a in "128 128 128" "256 256 256" "1024 1024 --batch 16" "2048 2048 --batch 16" "4096 4096 --batch 16"; do
  python profiles/pass_times.py $a >> gpurun_out/passes11.txt 2>&1
done
