"""Per-rank cost of the all-to-all distributed-FFT arm, measured on one GPU,
beside the halo slabs (SURVEY.md 8e comparison).

G engines of one process (pdgpu_set_transpose, rank r = engine r) run one
batched K.u of an N^2 lattice with device copies in place of the NCCL
transposes (pdgpu_group_matvec_transpose), all on this GPU: the total time is
the sum of the G ranks' compute plus the copies.  Per rank: t_total / G
(compute + pack/unpack, the copies included -- an upper bound for the rank's
work); the transposes move (G-1)/G of the rank's spectrum share twice per
K.u, converted to time at the NVLink 5 rate (900 GB/s per direction) for a
projected step = per-rank compute + transfer.  Efficiency = t_single /
(G * projected step).  usage: python tools/transpose_proj.py [N] [B] [G...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2301_11828_b200 import FastForce, build_kernel
    from paper_2301_11828_b200.engine import group_matvec_transpose, transpose_splits

    argv = sys.argv[1:]
    n = int(argv[0]) if len(argv) > 0 else 4096
    B = int(argv[1]) if len(argv) > 1 else 16
    Gs = [int(x) for x in argv[2:]] or [1, 2, 4, 8]
    h = 1.0 / n
    K = build_kernel(2, h, 3.015 * h, 3, 1.0, 1.0)
    u = torch.empty((B, 2, n, n), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    f = torch.empty_like(u)

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    single = FastForce((n, n), 3, K)
    single.set_geometry(h, [0.0, 0.0], 3.015 * h, 1.0)
    uf, ff = u.reshape(B, 2, -1), f.reshape(B, 2, -1)
    t_single = timed(lambda: single.matvec_device(uf, ff, B))
    single.close()
    out = {"n": n, "batch": B, "t_single_ms": t_single, "nvlink_gbs": 900.0, "runs": []}
    hx = n // 2 + 1
    for G in Gs:
        rb, cb = transpose_splits(n, n, G)
        engines = []
        for r in range(G):
            e = FastForce((n, rb[r + 1] - rb[r]), 3, K)
            e.set_geometry(h, [0.0, rb[r] * h], 3.015 * h, 1.0)
            e.set_transpose(G, r, n, rb, cb)
            engines.append(e)
        us = [u[:, :, rb[r]:rb[r + 1], :].contiguous().reshape(B, 2, -1) for r in range(G)]
        fs = [torch.empty_like(x) for x in us]
        t = timed(lambda: group_matvec_transpose(engines, us, fs, B), reps=3)
        # bytes a rank sends per K.u: two transposes of its spectrum share, the own block stays
        share = B * 2 * hx * (n // G) * 16
        sent = 2 * share * (G - 1) / G
        t_xfer = sent / 900e9 * 1e3
        per_rank = t / G
        proj = per_rank + t_xfer
        run = {"G": G, "t_group_ms": t, "per_rank_compute_ms": per_rank, "bytes_sent_per_rank": sent,
               "transfer_ms_at_900GBs": t_xfer, "projected_step_ms": proj,
               "projected_efficiency": t_single / (G * proj)}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
        for e in engines:
            e.close()
        del us, fs
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
