timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/trun.json 2> gpurun_out/trun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 3 --warmup 3 --shard slab > gpurun_out/trun_slab.json 2> gpurun_out/trun_slab.err
