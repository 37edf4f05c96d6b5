"""Per-pass times of one interior rank of a G-way halo-slab split (ghost rows
resident): python tools/slab_passes.py N B G [--dim 3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2301_11828_b200 import build_kernel
    from paper_2301_11828_b200.slab import SlabForce
    argv = list(sys.argv[1:])
    dim = 2
    if "--dim" in argv:
        i = argv.index("--dim")
        dim = int(argv[i + 1])
        del argv[i:i + 2]
    n, B, G = int(argv[0]), int(argv[1]), int(argv[2])
    M, h = 3, 1.0 / n
    K = build_kernel(dim, h, 3.015 * h, M, 1.0, 1.0)
    sf = SlabForce((n,) * dim, M, K, rank=G // 2, world=G, device=torch.device("cuda", 0), halo="ghost")
    sf.set_geometry(h, None, 3.015 * h, 1.0)
    ext, fext, g = sf._buf(B)
    ext.uniform_(-1, 1)
    g.uniform_(-1, 1)
    sf.eng.set_ghosts(g)
    s = torch.cuda.Stream()
    for _ in range(3):
        sf.eng.matvec_device(ext, fext, B, s)
    torch.cuda.synchronize()
    sf.eng.timing_read()
    sf.eng.timing(True)
    reps = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        sf.eng.matvec_device(ext, fext, B, s)
    b.record(s)
    torch.cuda.synchronize()
    print(f"n={n} dim={dim} B={B} G={G} rows={sf.L}: {a.elapsed_time(b) / reps:.4f} ms",
          {k: round(v[0] / reps, 4) for k, v in sf.eng.timing_read().items()})


if __name__ == "__main__":
    main()
