"""Per-rank cost of the halo-slab decomposition, measured on one GPU.

Builds the engine of one interior rank of a G-way row split of an N^2 lattice
(batch B) in both halo modes and times its K.u with CUDA events (ghost rows
resident: the NCCL exchange itself is not on this GPU), against the
single-GPU K.u of the whole lattice.  compute-only efficiency = t_single /
(G * t_rank).  Halo bytes per rank per step are reported beside it.
usage: python tools/slab_proj.py [N] [B] [G...] [--dim 3]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2301_11828_b200 import FastForce, build_kernel
    from paper_2301_11828_b200.slab import SlabForce

    argv = list(sys.argv[1:])
    dim = 2
    if "--dim" in argv:
        i = argv.index("--dim")
        dim = int(argv[i + 1])
        del argv[i:i + 2]
    n = int(argv[0]) if len(argv) > 0 else 4096
    B = int(argv[1]) if len(argv) > 1 else 16
    Gs = [int(x) for x in argv[2:]] or [2, 4, 8]
    M = 3
    h = 1.0 / n
    K = build_kernel(dim, h, 3.015 * h, M, 1.0, 1.0)
    dims = (n,) * dim
    nn = n ** dim
    plane = n ** (dim - 1)
    s = torch.cuda.Stream()

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    full = FastForce(dims, M, K)
    full.set_geometry(h, None, 3.015 * h, 1.0)
    u = torch.empty((B, dim, nn), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    f = torch.empty_like(u)
    t1 = timed(lambda: full.matvec_device(u, f, B, s))
    full.close()
    del u, f
    out = {"grid": list(dims), "batch": B, "single_gpu_ms": t1, "ranks": {}}
    for G in Gs:
        r = G // 2 if G > 1 else 0  # an interior rank
        row = {}
        for halo in ("ghost", "embedded"):
            sf = SlabForce(dims, M, K, rank=r, world=G, device=torch.device("cuda", 0), halo=halo)
            sf.set_geometry(h, None, 3.015 * h, 1.0)
            ext, fext, g = sf._buf(B)
            ext.uniform_(-1, 1)
            g.uniform_(-1, 1)
            if halo == "ghost":
                sf.eng.set_ghosts(g if G > 1 else None)
            t = timed(lambda: sf.eng.matvec_device(ext, fext, B, s))
            row[halo] = {"rank_ms": t, "engine_rows": sf.L, "embedding_bits": sf.eng.embedding(),
                         "compute_only_efficiency": t1 / (G * t)}
            sf.eng.close()
            del ext, fext, g
        # both directions of both interior faces: sent + received
        row["halo_bytes_per_rank_per_step"] = (2 if G > 2 else 1) * 2 * M * plane * dim * 8 * B if G > 1 else 0
        out["ranks"][str(G)] = row
    print(json.dumps(out))


if __name__ == "__main__":
    main()
