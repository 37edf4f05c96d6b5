"""The C++ drop-in header compiles against the reference's own types.

include/pdgpu.hpp is duck-typed on pdfast::Grid / Horizon / KernelStack /
VecField / Regions / BondLedger; this compiles a translation unit that uses it
exactly where the reference's call sites use FastForce and apply_corrections
(tests/test_corrections.cpp:320-323), with PDGPU_WITH_PDFAST error mapping,
and links it against libpdgpu.so.  Needs the reference tree (skipped on the
GPU box, where /root/reference does not exist)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj/include"

SRC = r"""
#include <fftw3.h>
#include "pdfast/convolution.hpp"
#include "pdfast/corrections.hpp"
#define PDGPU_WITH_PDFAST
#include "pdgpu.hpp"

int main() {
    using namespace pdfast;
    Grid<2> g; g.h = 0.0025; g.dims = {20, 20}; g.thickness = 0.0025;
    Horizon hz = Horizon::from_ratio(3, g.h);
    Material mat{2e11, 1.0 / 3.0, 7850.0, {}, {}, PlaneMode::Stress};
    auto K = build_kernel(g, hz, mat);
    auto regions = classify_regions<2>(g, hz, {});
    BondLedger ledger(g.n_nodes());
    ledger.break_bond(0, 1);
    VecField<2> u(g.n_nodes()), f(g.n_nodes());
    pdgpu::FastForce<2> engine(g, hz, K);          // was: FastForce<2> engine(g, hz, K);
    engine.apply(u, f);                              // same signature
    pdgpu::apply_corrections(engine, f, u, regions, ledger);
    return f.c[0].size() == 400 ? 0 : 1;
}
"""


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree absent")
def test_dropin_header_compiles_and_links(tmp_path):
    from paper_2301_11828_b200 import _lib
    lib = _lib.load()
    src = tmp_path / "dropin.cpp"
    src.write_text(SRC)
    exe = tmp_path / "dropin"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{REF}", f"-I{ROOT}/include", f"-I{ROOT}/oracle/fftw_cpu", str(src),
           os.path.join(ROOT, "oracle", "fftw_cpu", "fftw_cpu.cpp"), "-o", str(exe),
           f"-L{os.path.dirname(_lib.lib_path())}", "-lpdgpu", f"-Wl,-rpath,{os.path.dirname(_lib.lib_path())}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree absent")
def test_solver_level_dropin_compiles():
    """pdgpu::Simulation<Dim> (include/pdgpu_sim.hpp) against the reference's
    Problem / SolverOptions / SimState / BondLedger: the GPU test
    tests/test_gpu_cpp_dropin.py runs the resulting oracle/_ref/dropin_check."""
    cmd = ["g++", "-std=c++20", "-fsyntax-only", f"-I{REF}", f"-I{REF}/../tests", f"-I{ROOT}/include",
           f"-I{ROOT}/oracle/fftw_cpu", os.path.join(ROOT, "oracle", "dropin_check.cpp")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
