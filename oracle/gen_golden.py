"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  Runs here (where /root/reference exists and
oracle/_ref/libpdref.so was built from the unmodified reference headers +
oracle/fftw_cpu), never on the GPU box.  Every input is produced by the
reference's own generators (std::mt19937 through tests/support/oracles.hpp)
with the seeds of the reference's own tests; the fixtures keep only the
outputs plus input checksums, and tests/ regenerate the inputs with the C
restatement of the same RNG (oracle/oracle.c), which the checksums pin.

    python oracle/gen_golden.py            # writes tests/golden/*.npz
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path = [p for p in sys.path if os.path.abspath(p or ".") != HERE]
sys.path.insert(0, os.path.dirname(HERE))
from oracle.oracle import Oracle, RefProblem, Rng, _d, i64p, ip, rlib  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
STEEL_E = 2e11


def ref_random_kernel(rng: Rng, dim, M, h):
    np_ = dim * (dim + 1) // 2
    K = np.zeros((np_, (2 * M + 1) ** dim))
    rlib().ref_random_kernel(rng.h, dim, M, h, _d(K))
    return K


def ref_random_field(rng: Rng, dim, n, amp=1.0):
    u = np.zeros((dim, n))
    rlib().ref_random_field(rng.h, dim, n, amp, _d(u))
    return u


def ref_random_ledger(rng: Rng, dims, M, tries):
    import ctypes as C
    d = (C.c_int * len(dims))(*dims)
    out = np.zeros((tries + 1, 2), dtype=np.int64)
    n = rlib().ref_random_ledger(rng.h, len(dims), d, M, tries, out.ctypes.data_as(i64p), tries + 1)
    return out[:n]


def random_strip(rng: Rng, dims, h, M):
    """acceptance_main.cpp:43-59 random_strip, same rng call order."""
    dim = len(dims)
    axis = rng.next() % dim
    depth = (1 + rng.next() % M) * h
    lo = [0.0] * dim
    hi = [dims[d] * h for d in range(dim)]
    if rng.next() % 2:
        hi[axis] = lo[axis] + depth
    else:
        lo[axis] = hi[axis] - depth
    mask = 1 + (rng.next() % ((1 << dim) - 1))
    return lo, hi, mask


def pairs_hash(p):
    return hashlib.sha256(np.ascontiguousarray(p, dtype=np.int64).tobytes()).hexdigest()


def csum(a):
    a = np.asarray(a, dtype=np.float64)
    return np.array([a.sum(), (a * a).sum()])


def gen_conv():
    """tests/test_convolution.cpp:129-155 full-stack random-stencil cases."""
    out = {}
    for dim, shapes, bands in [(2, [(16, 12), (32, 32), (40, 20), (9, 7)], [2, 3, 4, 2]),
                               (3, [(8, 8, 8), (12, 10, 8), (16, 16, 16)], [2, 3, 4])]:
        rng = Rng(37 + dim, ref=True)
        for k, (dims, M) in enumerate(zip(shapes, bands)):
            h = 0.5
            K = ref_random_kernel(rng, dim, M, h)
            n = int(np.prod(dims))
            u = ref_random_field(rng, dim, n)
            r = RefProblem(dims, h=h, delta=M * h, M=M, E=1.0, thickness=1.0)
            r.set_stencils(K)
            r.finalize()
            tag = f"d{dim}_{k}"
            out[tag + "_dims"] = np.array(dims)
            out[tag + "_M"] = np.array(M)
            out[tag + "_K_csum"] = csum(K)
            out[tag + "_u_csum"] = csum(u)
            out[tag + "_f"] = r.apply(u)
            out[tag + "_resid"] = np.array(r.imag_residue())
            f_dir = np.zeros_like(u)
            rlib().ref_tbt_apply_all(r.h, _d(np.ascontiguousarray(u)), _d(f_dir))
            out[tag + "_fdirect"] = f_dir
    np.savez_compressed(os.path.join(OUT, "conv_random.npz"), **out)


def gen_corrections():
    """tests/test_corrections.cpp:301-338: strip constraint + 40 random bonds."""
    out = {}
    rng = Rng(1234, ref=True)
    for k, (dims, M) in enumerate([((20, 20), 3), ((16, 12), 2), ((40, 20), 4)]):
        h = 0.0025
        r = RefProblem(dims, h=h, delta=M * h, M=M, E=STEEL_E, thickness=0.0025)
        lo = (0.0, dims[1] * h - M * h)
        hi = (dims[0] * h, dims[1] * h)
        r.add_constraint(lo, hi, 0b01)
        led = ref_random_ledger(rng, dims, M, 40)
        for p, q in led:
            r.add_bond(int(p), int(q))
        u = ref_random_field(rng, 2, int(np.prod(dims)))
        r.finalize()
        tag = f"c{k}"
        out[tag + "_dims"] = np.array(dims)
        out[tag + "_M"] = np.array(M)
        out[tag + "_box"] = np.array(lo + hi)
        out[tag + "_ledger"] = r.ledger_pairs()
        out[tag + "_u_csum"] = csum(u)
        out[tag + "_f"] = r.matvec(u)
        out[tag + "_fdense"] = r.dense(u)
    np.savez_compressed(os.path.join(OUT, "corrections.npz"), **out)


def gen_acceptance():
    """acceptance_main.cpp:63-112 criteria 1/2: random strips, 0..50 bonds."""
    out = {}
    for dim, shapes in [(2, [(16, 12), (32, 32), (40, 20)]), (3, [(8, 8, 8), (12, 10, 8), (16, 16, 16)])]:
        rng = Rng(2024 + dim, ref=True)
        k = 0
        for dims in shapes:
            for M in (2, 3, 4):
                h = 0.01
                r = RefProblem(dims, h=h, delta=M * h, M=M, E=STEEL_E, thickness=0.0025)
                lo, hi, mask = random_strip(rng, dims, h, M)
                r.add_constraint(lo, hi, mask)
                nb = rng.next() % 51
                led = ref_random_ledger(rng, dims, M, nb)
                for p, q in led:
                    r.add_bond(int(p), int(q))
                u = ref_random_field(rng, dim, int(np.prod(dims)))
                r.finalize()
                tag = f"d{dim}_{k}"
                out[tag + "_dims"] = np.array(dims)
                out[tag + "_M"] = np.array(M)
                out[tag + "_box"] = np.array(list(lo) + list(hi))
                out[tag + "_mask"] = np.array(mask)
                out[tag + "_ledger"] = r.ledger_pairs()
                out[tag + "_u_csum"] = csum(u)
                out[tag + "_f"] = r.matvec(u)
                out[tag + "_fdense"] = r.dense(u)
                k += 1
    np.savez_compressed(os.path.join(OUT, "acceptance.npz"), **out)


def clamp_boxes(dim, d):
    boxes = []
    for ax in range(dim):
        lo0 = [0.0] * dim
        hi0 = [1.0] * dim
        hi0[ax] = d
        boxes.append((tuple(lo0), tuple(hi0)))
        lo1 = [0.0] * dim
        hi1 = [1.0] * dim
        lo1[ax] = 1.0 - d
        boxes.append((tuple(lo1), tuple(hi1)))
    return boxes


def config_problem(dims, ref=True):
    dim = len(dims)
    h = 1.0 / dims[0]
    d = 3.015 * h
    r = RefProblem(dims, h=h, delta=d, M=3, E=1.0, thickness=1.0)
    for lo, hi in clamp_boxes(dim, d):
        r.add_constraint(lo, hi, (1 << dim) - 1)
    r.finalize()
    return r


def gen_configs():
    """BASELINE configs 1 (128^2) and 4 (3D, shrunk to 24^3 for a fixture):
    delta = 3.015h clamped layers; K.u and the CG solve (new) over the
    reference mat-vec."""
    out = {}
    r = config_problem((128, 128))
    n = 128 * 128
    u = ref_random_field(Rng(1000, ref=True), 2, n)
    b = ref_random_field(Rng(1001, ref=True), 2, n)
    out["c1_u_csum"] = csum(u)
    out["c1_f"] = r.matvec(u)
    x, it, rel, hist = r.cg(b, tol=1e-10, maxit=20000, nhist=20)
    out["c1_cg_iters"] = np.array(it)
    out["c1_cg_relres"] = np.array(rel)
    out["c1_cg_x"] = x
    out["c1_cg_x20"] = hist[19]
    r3 = config_problem((24, 24, 24))
    u3 = ref_random_field(Rng(4000, ref=True), 3, 24 ** 3)
    out["c4_u_csum"] = csum(u3)
    out["c4_f"] = r3.matvec(u3)
    np.savez_compressed(os.path.join(OUT, "configs.npz"), **out)


def gen_seeds():
    """Crack seeding of BASELINE configs 3 and 5 (fracture.hpp:164-198)."""
    out = {}
    for tag, n, seg in [("c3", 1024, ((0.25, 0.5), (0.75, 0.5))), ("c5", 2048, ((0.0, 0.5), (0.25, 0.5)))]:
        h = 1.0 / n
        r = RefProblem((n, n), h=h, delta=3.015 * h, M=3, E=1.0, thickness=1.0)
        r.add_segment(seg[0], seg[1], 0.0)
        r.finalize()
        p = r.ledger_pairs()
        out[tag + "_count"] = np.array(len(p))
        out[tag + "_first"] = p[:64]
        out[tag + "_hash"] = np.array(pairs_hash(p))
    np.savez_compressed(os.path.join(OUT, "seeds.npz"), **out)


def precracked_problem():
    """preset("precracked_plate", 0.05/100) as acceptance_main.cpp:197-219 uses it
    (scenario.hpp:515-538): 100x100, velocity-driven top/bottom layers, s0 = 0.01."""
    h = 0.05 / 100.0
    delta = 3 * h
    r = RefProblem((100, 100), h=h, delta=delta, M=3, E=2e11, thickness=0.0025, rho=7850.0)
    r.add_constraint((0.0, 0.05 - delta), (0.05, 0.05), 0b10, 1, 20.0)
    r.add_constraint((0.0, 0.0), (0.05, delta), 0b10, 1, -20.0)
    r.add_segment((0.02, 0.025), (0.03, 0.025), 0.0)
    r.finalize()
    return r


def gen_vv():
    """Criterion 5 trajectory: 200 velocity-Verlet steps with bond breaking."""
    out = {}
    # s0 = 0.01 is the preset (no bond breaks in 200 steps); s0 = 5e-3 makes
    # the velocity layers tear progressively (88 distinct breaking steps)
    for tag, s0 in (("s0_1e-2", 0.01), ("s0_5e-3", 5e-3)):
        r = precracked_problem()
        r.sim_init(1.3367e-8, s0=s0)
        per_step = []
        for _ in range(200):
            per_step.append(r.sim_step(1))
        u, v, f, t = r.sim_get()
        out.update({tag + "_u": u, tag + "_v": v, tag + "_t": np.array(t),
                    tag + "_broken_per_step": np.array(per_step, dtype=np.int64), tag + "_ledger": r.ledger_pairs()})
    np.savez_compressed(os.path.join(OUT, "vv_precracked.npz"), **out)


def snapshot_case(dim):
    """Fields of the snapshot goldens: mt19937 values (seed 6000 + dim) scaled
    over many decades, plus exact edge values (0, -0, 1/3, tiny, huge)."""
    dims = (7, 5) if dim == 2 else (4, 3, 2)
    n = int(np.prod(dims))
    rng = Rng(6000 + dim, ref=True)
    u = rng.uniform(dim * n).reshape(dim, n) * 10.0 ** np.linspace(-300, 300, dim * n).reshape(dim, n)
    u[0, :5] = [0.0, -0.0, 1.0 / 3.0, 5e-324, 1.7976931348623157e308]
    damage = rng.uniform(n) * 0.5 + 0.5
    origin = np.array([0.125, -2.0 / 3.0, 1e-17][:dim])
    return dims, 1.0 / 1024.0 if dim == 2 else 0.1, origin, u, damage, 42 if dim == 2 else 1234567, 0.1 * 3


def gen_snapshots():
    """Snapshot files written by the reference's write_snapshot_dat (output.hpp:76-102),
    run through oracle/_ref/snap_writer on raw fp64 inputs."""
    import subprocess
    import tempfile
    exe = os.path.join(HERE, "_ref", "snap_writer")
    for dim in (2, 3):
        dims, h, origin, u, damage, step, t = snapshot_case(dim)
        d = os.path.join(OUT, f"snap{dim}d")
        with tempfile.TemporaryDirectory() as tmp:
            fu, fd = os.path.join(tmp, "u.raw"), os.path.join(tmp, "d.raw")
            np.ascontiguousarray(u).tofile(fu)
            np.ascontiguousarray(damage).tofile(fd)
            args = [exe, str(dim), *map(str, dims), repr(h), *map(repr, origin.tolist()), str(step), repr(t), d, fu, fd]
            subprocess.run(args, check=True, capture_output=True)


def monitor_case(dim):
    """Inputs of the monitor goldens: a small lattice, monitor points inside,
    on node coordinates, between nodes and outside the domain (clamped), and
    rows whose fields hold edge values (+-0, subnormal, huge) at those nodes."""
    dims = (10, 10) if dim == 2 else (4, 3, 2)
    h = 0.01 if dim == 2 else 0.1
    origin = np.array([0.0, 0.0, 0.0][:dim]) if dim == 2 else np.array([0.125, -2.0 / 3.0, 1e-17])
    if dim == 2:
        pts = np.array([[0.055, 0.025], [0.0, 0.0], [0.1, 0.1], [-1.0, 0.05], [0.0999999, 2.0], [0.03, 0.07]])
    else:
        pts = origin + np.array([[0.05, 0.05, 0.05], [0.3, 0.2, 0.1], [-5.0, 9.0, 0.15], [0.1, 0.1, 0.0999999999]])
    n = int(np.prod(dims))
    rng = Rng(7000 + dim, ref=True)
    steps = [0, 12, 9999999]
    ts = [0.0, 12 * 2e-8, 1.0 / 3.0]
    rows = []
    for r in range(3):
        u = rng.uniform(dim * n).reshape(dim, n) * 10.0 ** np.linspace(-200, 200, dim * n).reshape(dim, n)
        u[:, :4] = [[0.0, -0.0, 5e-324, 1.7976931348623157e308]] * dim
        u[0, n - 1] = 3.5e-5
        rows.append((steps[r], ts[r], u))
    return dims, h, origin, pts, rows


def gen_monitors():
    """Monitor files written by the reference's MonitorWriter (output.hpp:45-72)
    through oracle/_ref/snap_writer, plus the inputs and the nodes it chose."""
    import subprocess
    import tempfile
    exe = os.path.join(HERE, "_ref", "snap_writer")
    out = {}
    for dim in (2, 3):
        dims, h, origin, pts, rows = monitor_case(dim)
        path = os.path.join(OUT, f"monitor{dim}d.tsv")
        with tempfile.TemporaryDirectory() as tmp:
            fp, fr = os.path.join(tmp, "p.raw"), os.path.join(tmp, "r.raw")
            np.ascontiguousarray(pts, dtype=np.float64).tofile(fp)
            np.concatenate([np.concatenate([[s, t], u.ravel()]) for s, t, u in rows]).tofile(fr)
            args = [exe, "mon", str(dim), *map(str, dims), repr(h), *map(repr, origin.tolist()), path, fp,
                    str(len(pts)), fr, str(len(rows))]
            res = subprocess.run(args, check=True, capture_output=True, text=True)
        out[f"nodes{dim}d"] = np.array([int(x) for x in res.stdout.split()], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "monitor_nodes.npz"), **out)


def adr_problem(dims, ref=True):
    """Quasi-static plate/cube for the reference's ADR solver (timestepping.hpp:79-162):
    bottom layer clamped, a downward load on the top layer."""
    dim = len(dims)
    h = 1.0 / dims[0]
    d = 3.015 * h
    P = RefProblem(dims, h=h, delta=d, M=3, E=1.0, thickness=1.0) if ref else \
        Oracle(dims, h=h, delta=d, M=3, E=1.0, thickness=1.0)
    lo, hi = [0.0] * dim, [1.0] * dim
    hi[dim - 1] = d
    P.add_constraint(lo, hi, (1 << dim) - 1)
    llo, lhi = [0.0] * dim, [1.0] * dim
    llo[dim - 1] = 1.0 - d
    val = [0.0] * dim
    val[dim - 1] = -1e-3
    P.add_load(llo, lhi, val)
    if ref:
        P.finalize()
    return P


ADR_CASES = (("p2", (64, 64), None, 300), ("p2_fixed", (64, 64), 0.05, 200), ("p3", (16, 16, 16), None, 100))


def gen_adr():
    """ADR trajectories (adaptive and fixed damping): u, v_half-driven damping
    trace every 25 steps."""
    out = {}
    for tag, dims, fixed, steps in ADR_CASES:
        r = adr_problem(dims)
        r.sim_init_adr(1.0, fixed_damping=fixed)
        trace = []
        for k in range(steps // 25):
            r.sim_step(25)
            trace.append(r.adr_damping())
        u, v, f, t = r.sim_get()
        out.update({tag + "_u": u, tag + "_f": f, tag + "_t": np.array(t), tag + "_damping": np.array(trace)})
    np.savez_compressed(os.path.join(OUT, "adr.npz"), **out)


def main():
    os.makedirs(OUT, exist_ok=True)
    fns = {"conv": gen_conv, "corrections": gen_corrections, "acceptance": gen_acceptance, "configs": gen_configs,
           "seeds": gen_seeds, "vv": gen_vv, "snapshots": gen_snapshots, "monitors": gen_monitors, "adr": gen_adr}
    pick = sys.argv[1:] or list(fns)
    for name in pick:
        fns[name]()
        print("wrote", name)


if __name__ == "__main__":
    main()
