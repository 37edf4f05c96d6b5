"""Config 5 pull-rate scan (BASELINE configs[4]): 2048^2 plate, notch L/4 at
the left edge midline, velocity-driven top/bottom delta layers (+-v), s0 = 1e-3,
velocity Verlet at dt = 0.8 x the Gershgorin-stable step, 2000 steps.  For each
rate: bonds broken per 100 steps, the crack-tip x (furthest broken bond within
0.05 of the midline) and the bonds broken next to the loaded layers.

    python tools/crack_scan.py [--n 2048] [--steps 2000] [--rates 1e-4,3e-4,...]
    rate suffix 's' = displacement per step (v = rate / dt)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--chunk", type=int, default=100)
    ap.add_argument("--rates", default="1e-4,3e-4,1e-3,1e-4s")
    a = ap.parse_args()
    from paper_2301_11828_b200 import FastForce, build_kernel
    n = a.n
    h = 1.0 / n
    dl = 3.015 * h
    M = 3
    K = build_kernel(2, h, dl, M, 1.0, 1.0)
    lam = max(sum(2.0 * np.abs(K[0 if (x, y) == (0, 0) else (1 if x != y else 2)]).sum() for y in range(2))
              for x in range(2))
    dt = 0.8 * 2.0 * (1.0 / lam) ** 0.5
    out = {"grid": [n, n], "dt": dt, "s0": 1e-3, "steps": a.steps, "runs": []}
    for rs in a.rates.split(","):
        per_step = rs.endswith("s")
        rate = float(rs.rstrip("s"))
        v = rate / dt if per_step else rate
        ff = FastForce((n, n), M, K, device=0)
        ff.set_geometry(h, [0.0, 0.0], dl, 1.0)
        ff.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1, v)
        ff.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 1, -v)
        notch = ff.seed_segment((0.0, 0.5), (0.25, 0.5))
        ff.sim_init(dt)
        hist = []
        t0 = time.time()
        done = 0
        while done < a.steps:
            k = min(a.chunk, a.steps - done)
            nb = ff.sim_step(k, 1e-3)
            done += k
            hist.append(int(nb))
        wall = time.time() - t0
        pairs = ff.ledger_pairs()
        ok = ff.sim_finite()
        ff.close()
        p, q = pairs[:, 0], pairs[:, 1]
        xm = ((p % n) + (q % n)) * 0.5 * h
        ym = ((p // n) + (q // n)) * 0.5 * h
        mid = np.abs(ym - 0.5) < 0.05
        tip = float(xm[mid].max()) if mid.any() else None
        edge = int(((ym < 0.05) | (ym > 0.95)).sum())
        run = {"rate": rs, "v": v, "notch_bonds": notch, "broken_total": int(len(pairs)),
               "broken_per_chunk": hist, "chunk": a.chunk, "crack_tip_x": tip, "edge_bonds": edge,
               "finite": ok, "wall_s": wall}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
