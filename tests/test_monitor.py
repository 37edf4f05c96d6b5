"""MonitorWriter (output.hpp:45-72) through libpdgpu's host writer: the golden
files were written by the reference's own MonitorWriter (oracle/snap_writer.cpp
"mon" mode via oracle/gen_golden.py) from small lattices with monitor points
inside, on, between and outside the nodes, and fields holding edge values at
the monitored nodes.  Our nodes must equal the reference's nearest_node
choice and the files must match byte for byte; an unwritable path raises
IoError like the reference (tests/test_output.cpp:115-117).  The GPU test
records rows during sim_step on the device and checks them against the
field read back after every step."""
import os
import sys

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, os.path.dirname(GOLD).rsplit(os.sep, 1)[0])


@pytest.mark.parametrize("dim", [2, 3])
def test_monitor_matches_reference_bytes(dim, tmp_path):
    from oracle.gen_golden import monitor_case
    from paper_2301_11828_b200 import MonitorWriter
    dims, h, origin, pts, rows = monitor_case(dim)
    ref_nodes = np.load(os.path.join(GOLD, "monitor_nodes.npz"))[f"nodes{dim}d"]
    path = str(tmp_path / "monitor.tsv")
    mon = MonitorWriter(path, dims, h, origin, pts)
    assert np.array_equal(mon.nodes, ref_nodes)
    for step, t, u in rows:
        mon.append(step, t, u)
    mon.close()
    assert open(path, "rb").read() == open(os.path.join(GOLD, f"monitor{dim}d.tsv"), "rb").read()


def test_monitor_reference_unit_case(tmp_path):
    """tests/test_output.cpp:80-118 restated: node lin(5, 2), full-precision row, clamping."""
    from paper_2301_11828_b200 import MonitorWriter
    path = str(tmp_path / "monitor.tsv")
    mon = MonitorWriter(path, (10, 10), 0.01, (0.0, 0.0), [(0.055, 0.025)])
    assert list(mon.nodes) == [2 * 10 + 5]
    u = np.zeros((2, 100))
    u[0, mon.nodes[0]] = 3.5e-5
    mon.append(12, 12 * 2e-8, u)
    mon.close()
    head, row = open(path).read().splitlines()[:2]
    assert "u_x" in head
    c = row.split("\t")
    assert int(c[0]) == 12 and int(c[2]) == mon.nodes[0] + 1 and float(c[3]) == 3.5e-5 and float(c[4]) == 0.0
    corner = MonitorWriter("", (10, 10), 0.01, (0.0, 0.0), [(0.0, 0.0), (0.1, 0.1)])
    assert list(corner.nodes) == [0, 99]


def test_monitor_unwritable_path_raises():
    from paper_2301_11828_b200 import IoError, MonitorWriter
    with pytest.raises(IoError):
        MonitorWriter("/nonexistent_dir/m.tsv", (10, 10), 0.01, (0.0, 0.0), [(0.05, 0.05)])


@pytest.mark.gpu
def test_sim_monitor_rows_on_device(tmp_path):
    from paper_2301_11828_b200 import FastForce, MonitorWriter, build_kernel
    n = 64
    h = 1.0 / n
    dl = 3.015 * h
    ff = FastForce((n, n), 3, build_kernel(2, h, dl, 3, 1.0, 1.0), device=0)
    ff.set_geometry(h, [0.0, 0.0], dl, 1.0)
    ff.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1, 1e-3)
    ff.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 1, -1e-3)
    ff.sim_init(1e-3)
    pts = [(0.5, 0.9), (0.25, 0.75), (0.5, 0.5)]
    path = str(tmp_path / "m.tsv")
    mon = MonitorWriter(path, (n, n), h, (0.0, 0.0), pts)
    ff.sim_monitor(mon.nodes)
    ref = MonitorWriter(str(tmp_path / "r.tsv"), (n, n), h, (0.0, 0.0), pts)
    for k in range(7):  # one step per call: the host field of every step for the check
        ff.sim_step(1)
        u, _, _, t = ff.sim_get()
        ref.append(k + 1, t, u)  # State::step after the step (tools/pdfast_cli.cpp:76)
    assert mon.append_sim(ff) == 7
    ff.sim_step(5000)  # past the device row buffer (spill to host)
    steps, ts, vals = ff.sim_monitor_read()
    assert len(steps) == 5000 and steps[0] == 8 and steps[-1] == 5007
    u, _, _, t = ff.sim_get()
    assert np.array_equal(vals[-1], u[:, mon.nodes].T) and ts[-1] == t
    mon.close()
    ref.close()
    assert open(path, "rb").read() == open(str(tmp_path / "r.tsv"), "rb").read()
    ff.close()

