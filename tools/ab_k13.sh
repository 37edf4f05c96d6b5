# A/B of the K1 early row fetch and the K3 landed-operand variants (4096^2 x 16)
# usage (GPU box): bash tools/ab_k13.sh > gpurun_out/ab_k13.txt 2>&1
T="python -m pytest tests/test_gpu_scale.py -q -x -k test_config2_4096_matvec"
P="python profiles/pass_times.py 4096 4096 --batch 16 --reps 10"
for v in "PDGPU_K1_EARLY=0" "PDGPU_K1_EARLY=1" "PDGPU_K3=tx" "PDGPU_K3=tx2"; do
  echo "== $v"
  env $v $T 2>&1 | tail -1
  env $v $P 2>&1 | tail -1
  env $v $P 2>&1 | tail -1
done
echo "== 2048 (lq 11) tx"; PDGPU_K3=tx python profiles/pass_times.py 2048 2048 --batch 16 --reps 10 | tail -1
PDGPU_K3=tx python -m pytest tests/test_gpu_embedding.py tests/test_gpu_matvec.py -q -x 2>&1 | tail -1
echo "== 2048 base"; python profiles/pass_times.py 2048 2048 --batch 16 --reps 10 | tail -1
