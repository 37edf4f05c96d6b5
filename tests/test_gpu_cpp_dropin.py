"""The C++ drop-in executed on the GPU beside the reference's own C++ path.

oracle/_ref/dropin_check (oracle/dropin_check.cpp) is compiled in the build
container against the unmodified reference headers and libpdgpu.so, and runs
here on the reference's own types:

  matvec_2d / matvec_3d   pdgpu::FastForce<Dim>::apply + pdgpu::apply_corrections
                          vs pdfast::FastForce::apply + apply_corrections <= 1e-11
  update_bonds            pdgpu::update_bonds vs pdfast::update_bonds: same pairs,
                          same order, BondLedger::operator== (ledger.hpp:44)
  simulation_vv_fracture  pdgpu::Simulation<2> vs pdfast::Simulation<2> on the
                          criterion-5 problem, 200 steps: newly_broken() equal every
                          step, ledgers equal, u within 1e-8 (acceptance_main.cpp:197-219)
  simulation_adr          Integrator::Adr, 60 steps, u and damping within 1e-9
  evaluate_force_and_cg   Simulation::evaluate_force <= 1e-11; solve_static's
                          solution meets 1e-10 through the reference's operator
  exceptions              HorizonTooLargeForGrid, ShapeMismatch, LedgerOutOfBand
  monitor                 pdgpu::MonitorWriter on device-recorded rows vs the reference
                          MonitorWriter fed every step: nodes, steps, t equal, u <= 1e-8
"""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_check")
CHECKS = {"matvec_2d", "matvec_3d", "update_bonds", "simulation_vv_fracture", "simulation_adr",
          "evaluate_force_and_cg", "exceptions", "monitor"}


@pytest.fixture(scope="module")
def results():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/dropin_check not built (needs the reference tree at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    out = {}
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            d = json.loads(line)
            out[d["check"]] = d
    assert set(out) == CHECKS, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    return out


@pytest.mark.parametrize("name", sorted(CHECKS))
def test_dropin(results, name):
    assert results[name]["pass"], results[name]
