"""Pins of the oracle's Philox4x32-10 and Brownian-increment map (DESIGN.md pin H0; R8).

The oracle's generator is checked against (i) published known-answer vectors,
(ii) the CUDA toolkit's own curand_Philox4x32_10 evaluated on the host (an
independent implementation), and (iii) distributional statistics.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest
from scipy import stats

from oracle import philox

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat():
    rows = []
    with open(os.path.join(HERE, "golden", "philox_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([int(t, 16) for t in line.split()])
    return rows


def test_philox_known_answers():
    for row in _kat():
        out = philox.philox4x32_10(*row[:6])
        assert [int(x) for x in out] == row[6:], row


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path_factory.mktemp("pch") / "pch")
    subprocess.run([nvcc, "-O2", "-Wno-deprecated-gpu-targets", "-o", exe,
                    os.path.join(HERE, "tools", "philox_curand_host.cu")], check=True)
    return exe


def test_philox_matches_curand_host(curand_host):
    rng = np.random.default_rng(1234)
    ctr = rng.integers(0, 2 ** 32, size=(500, 6), dtype=np.uint64)
    ctr[:50, 4:] = 0                            # seed 0 keys, as in every config
    ctr[50:100, 3] = philox.INIT_STREAM
    inp = "\n".join(" ".join("%x" % v for v in row) for row in ctr) + "\n"
    out = subprocess.run([curand_host], input=inp, capture_output=True, text=True, check=True)
    ref = np.array([[int(t, 16) for t in l.split()] for l in out.stdout.strip().split("\n")])
    for i, row in enumerate(ctr):
        got = [int(x) for x in philox.philox4x32_10(*[int(v) for v in row])]
        assert got == list(ref[i]), (i, row)
    # vectorised path agrees with the scalar path
    k0, k1 = 0x1234, 0x9876
    v = philox.philox4x32_10(ctr[:, 0], ctr[:, 1], ctr[:, 2], ctr[:, 3], k0, k1)
    for i in (0, 17, 499):
        s = philox.philox4x32_10(*[int(x) for x in ctr[i, :4]], k0, k1)
        assert [int(a[i]) for a in v] == [int(b) for b in s]


def test_unit_map_exact_and_open_interval():
    x = np.array([0, 1, 511, 512, 2 ** 31, 2 ** 32 - 1], dtype=np.uint32)
    u = philox.uint_to_unit(x)
    assert u.min() > 0.0 and u.max() < 1.0
    # exact in float32: the float32 rounding of u is u itself (R8)
    assert np.all(u.astype(np.float32).astype(np.float64) == u)
    assert u[0] == 2.0 ** -24 and u[-1] == 1.0 - 2.0 ** -24


def test_normals_statistics():
    """mean within 4·sqrt(Δt/K), variance within 2%, plus a KS test."""
    d, dt = 100, 1.0 / 20
    dw = philox.brownian_increments(0, 3, 7, np.arange(10000), d, dt)   # K = 1e6
    K = dw.size
    assert abs(dw.mean()) < 4.0 * np.sqrt(dt / K)
    assert abs(dw.var() / dt - 1.0) < 0.02
    z = dw.ravel() / np.sqrt(dt)
    assert stats.kstest(z[:200000], "norm").pvalue > 1e-4
    # components are uncorrelated across the 4-block boundary and within it
    c = np.corrcoef(dw[:, :8].T)
    assert np.max(np.abs(c - np.eye(8))) < 0.05


def test_normals_deterministic_and_shard_invariant():
    """S:295 determinism; S:336 'path m depends only on (seed, m)'."""
    a = philox.standard_normals(5, 2, 3, np.arange(64), 13)
    b = philox.standard_normals(5, 2, 3, np.arange(64), 13)
    assert np.array_equal(a, b)
    c = np.vstack([philox.standard_normals(5, 2, 3, np.arange(32), 13),
                   philox.standard_normals(5, 2, 3, np.arange(32, 64), 13)])
    assert np.array_equal(a, c)
    # different step / iteration / seed give different draws
    assert not np.allclose(a, philox.standard_normals(5, 2, 4, np.arange(64), 13))
    assert not np.allclose(a, philox.standard_normals(5, 3, 3, np.arange(64), 13))
    assert not np.allclose(a, philox.standard_normals(6, 2, 3, np.arange(64), 13))
    # the first d components do not depend on d (ragged 4-blocks)
    assert np.array_equal(a[:, :10], philox.standard_normals(5, 2, 3, np.arange(64), 10))


def test_init_uniforms_in_range():
    u = philox.init_uniforms(0, 7, 1001)
    assert u.shape == (1001,) and u.min() > 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 0.05
