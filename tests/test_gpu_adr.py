"""GPU ADR (AdrIntegrator, timestepping.hpp:79-162) against the CPU oracle and
the reference's own trajectories (tests/golden/adr.npz, oracle/gen_golden.py):
after the full run max|du| <= 1e-8 max|u| (the reference's own FFT-vs-dense
ADR criterion, tests/test_timestepping.cpp:168-176) and the damping trace to
1e-6; step for step over the first 50 steps u to 1e-11 relative L2."""
import os

import numpy as np
import pytest

from oracle.gen_golden import ADR_CASES, adr_problem

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def gpu_problem(dims):
    from paper_2301_11828_b200 import FastForce
    o = adr_problem(dims, ref=False)
    dim = len(dims)
    h = 1.0 / dims[0]
    d = 3.015 * h
    ff = FastForce(dims, 3, o.kernel())
    ff.set_geometry(h, [0.0] * dim, d, 1.0)
    lo, hi = [0.0] * dim, [1.0] * dim
    hi[dim - 1] = d
    ff.add_constraint(lo, hi, (1 << dim) - 1)
    llo, lhi = [0.0] * dim, [1.0] * dim
    llo[dim - 1] = 1.0 - d
    val = [0.0] * dim
    val[dim - 1] = -1e-3
    ff.add_load(llo, lhi, val)
    return o, ff


@pytest.mark.parametrize("tag,dims,fixed,steps", ADR_CASES)
def test_adr_matches_reference(tag, dims, fixed, steps):
    g = np.load(os.path.join(G, "adr.npz"))
    o, ff = gpu_problem(dims)
    ff.sim_init_adr(1.0, fixed_damping=fixed)
    trace = []
    for _ in range(steps // 25):
        ff.sim_step(25)
        trace.append(ff.adr_damping())
    u, v, f, t = ff.sim_get()
    assert t == float(g[tag + "_t"])
    # the reference's own FFT-vs-dense ADR criterion (tests/test_timestepping.cpp:168-176)
    assert np.abs(u - g[tag + "_u"]).max() <= 1e-8 * np.abs(g[tag + "_u"]).max()
    assert np.allclose(trace, g[tag + "_damping"], rtol=1e-6, atol=0)
    # and the oracle restatement, step for step over the first 50 steps
    o2, ff2 = gpu_problem(dims)
    o2.sim_init_adr(1.0, fixed_damping=fixed)
    ff2.sim_init_adr(1.0, fixed_damping=fixed)
    for k in range(50):
        o2.sim_step(1)
        ff2.sim_step(1)
        if k % 10 == 9:
            uo = o2.sim_get()[0]
            ug = ff2.sim_get()[0]
            assert np.linalg.norm(ug - uo) <= 1e-11 * max(np.linalg.norm(uo), 1e-300)
            assert abs(ff2.adr_damping() - o2.adr_damping()) <= 1e-9 * max(abs(o2.adr_damping()), 1e-300)


def test_adr_then_vv_reinit():
    """sim_init after an ADR run returns to velocity Verlet (Integrator::Vv)."""
    o, ff = gpu_problem((32, 32))
    ff.sim_init_adr(1.0)
    ff.sim_step(5)
    ff.sim_init(1e-3)
    o.sim_init(1e-3)
    ff.sim_step(5)
    o.sim_step(5)
    assert np.linalg.norm(ff.sim_get()[0] - o.sim_get()[0]) <= 1e-11 * np.linalg.norm(o.sim_get()[0])
