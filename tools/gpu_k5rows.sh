for tr in 1 2 4 8; do
  for a in "1024 1024 --batch 16" "2048 2048 --batch 16"; do
    echo "TR=$tr $(PDGPU_K5_ROWS=$tr python profiles/pass_times.py $a 2>&1)" >> gpurun_out/k5rows.txt
  done
done
