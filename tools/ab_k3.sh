# A/B of the K3 variants at 4096^2 x 16 (GPU box)
T="python -m pytest tests/test_gpu_scale.py -q -x -k test_config2_4096_matvec"
P="python profiles/pass_times.py 4096 4096 --batch 16 --reps 10"
for v in ${AB_VARIANTS:-"PDGPU_K3=tm PDGPU_K3=tx PDGPU_K3=tx3"}; do
  echo "== $v"
  env $v $T 2>&1 | tail -1
  env $v $P 2>&1 | tail -1
  env $v $P 2>&1 | tail -1
done
