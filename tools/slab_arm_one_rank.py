"""bench.run_slab with a single rank (the N > 1 arm's code path on one GPU):
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 tools/slab_arm_one_rank.py"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    sys.exit(bench.run_slab(argparse.Namespace(steps=5, warmup=3, no_e2e=False, no_cpu=True, no_extra=True)))
