"""`#moesim-report v1` writer (paper_2505_13345_b200/report.py): the double
formatting matches std::to_chars (the reference's format_double, io.cpp:55-60)
bit for bit; the bounds/metrics restatements match the reference's rules."""
import os
import struct
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2505_13345_b200 import report as R

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def to_chars():
    exe = os.path.join(tempfile.mkdtemp(), "to_chars_probe")
    subprocess.run(["g++", "-std=c++20", "-O1", "-o", exe, os.path.join(HERE, "cpp", "to_chars_probe.cpp")],
                   check=True)

    def run(vals):
        inp = "\n".join(struct.unpack("<Q", struct.pack("<d", v))[0].to_bytes(8, "big").hex() for v in vals) + "\n"
        return subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.splitlines()
    return run


def test_format_double_matches_to_chars(to_chars):
    rng = np.random.default_rng(0)
    vals = [0.0, -0.0, 1.0, 0.5, 2.0 / 3.0, 1e-5, 1e-4, 123456.0, 1234567.0, 1e15, 1e16, 1e17, 1e20, 1e21, 1e22,
            12345678901234567890.0, 5e-324, 1.7976931348623157e308, 0.1, 0.30000000000000004, 4.0 / 3.0, 2.0,
            1.5, 100.0, 1e100, 3.14159, 0.001, 0.000123]
    vals += list(rng.uniform(-1, 1, 200)) + list(10.0 ** rng.uniform(-30, 30, 200)) + \
        list(np.round(rng.uniform(0, 1e6, 100))) + list(rng.integers(0, 10 ** 9, 50).astype(float) / 64.0)
    want = to_chars(vals)
    got = [R.format_double(v) for v in vals]
    bad = [(v, g, w) for v, g, w in zip(vals, got, want) if g != w]
    assert not bad, bad[:5]


def test_replica_bounds_rule():
    # test_collab.cpp:108-203: (8, 64, 4) -> [1, 4], (2, 8, 8) -> [2, 2]
    assert R.replica_bounds(8, 64, 4) == (1.0, 4.0)
    assert R.replica_bounds(2, 8, 8) == (2.0, 2.0)


def test_intra_inter_metrics_order():
    p = np.arange(16, dtype=float).reshape(4, 4) / 15.0
    intra, inter = R.intra_inter_metrics(p, [[0, 1], [3, 2]])
    assert intra[0] == (p[0, 1] + p[1, 0]) / 2.0
    assert inter[(0, 1)] == (p[0, 3] + p[0, 2] + p[1, 3] + p[1, 2]) / 4.0


def test_report_writer_layout():
    w = R.ReportWriter()
    w.kv("command", "simulate")
    w.kv("replicas.mean", 1.5)
    w.kv("bytes.cross_device", 32)
    assert w.text() == "#moesim-report v1\ncommand=simulate\nreplicas.mean=1.5\nbytes.cross_device=32\n"
