"""Snapshot files (output.hpp:74-154) through libpdgpu's host writer/reader:
the golden files were written by the reference's own write_snapshot_dat
(oracle/snap_writer.cpp via oracle/gen_golden.py) from edge-case fields
(+-0, subnormal, DBL_MAX, values across 600 decades).  Reading a golden file
must give exactly the numbers Python parses from it, and writing those
numbers back must reproduce the file byte for byte."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _parse(path, dim):
    head, rows = {}, []
    for line in open(path):
        if line.startswith("#"):
            k, *v = line[1:].split()
            head[k] = v
        elif line.strip():
            rows.append([float(x) for x in line.split()[1:]])
    a = np.array(rows)
    return head, a[:, :dim].T.copy(), a[:, dim].copy()


@pytest.mark.parametrize("dim,name", [(2, "snap2d/snap_0000042.dat"), (3, "snap3d/snap_1234567.dat")])
def test_snapshot_roundtrip_matches_reference_bytes(dim, name, tmp_path):
    from paper_2301_11828_b200.engine import read_snapshot, write_snapshot
    path = os.path.join(GOLD, name)
    head, u_py, d_py = _parse(path, dim)
    snap = read_snapshot(path, dim)
    assert snap["dims"] == tuple(int(x) for x in head["dims"])
    assert snap["step"] == int(head["step"][0])
    assert np.array_equal(snap["u"].view(np.uint64), u_py.view(np.uint64))  # bit-exact, incl. -0
    assert np.array_equal(snap["damage"].view(np.uint64), d_py.view(np.uint64))
    out = write_snapshot(str(tmp_path), snap["dims"], snap["h"], snap["origin"], snap["u"], snap["step"], snap["t"],
                         snap["damage"])
    assert os.path.basename(out) == os.path.basename(path)
    assert open(out, "rb").read() == open(path, "rb").read()


def test_snapshot_bad_file(tmp_path):
    from paper_2301_11828_b200.engine import read_snapshot
    p = tmp_path / "bad.dat"
    p.write_text("# dims 2 2\n9 1 2 3\n")
    with pytest.raises(ValueError):
        read_snapshot(str(p), 2)
