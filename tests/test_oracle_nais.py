"""Pins of the NAIS-Net per-step oracle (oracle/nais.py).

N1 central finite differences of the hand adjoint (incl. R̄ = -R(Ā + Āᵀ));
N2 A = -RᵀR - εI is symmetric negative definite (SPEC nets invariants and
examples); N3 the Frobenius projection (examples, idempotence, monotonicity);
N4 with R = B = C = 0 the block is the identity on H1 ≥ 0, so the loss equals
the independently pinned residual-block oracle (bsde.py) with W2 = b2 = 0;
N5 initialisation.
"""
import numpy as np
import pytest

from oracle import bsde, nais


def _params(seed, d, w, N, scale=0.2):
    p = nais.init_params(seed, d, w, N)
    return p + scale * np.random.default_rng(seed).standard_normal(p.size)


@pytest.mark.parametrize("problem", [bsde.HEAT, bsde.HJB, bsde.ALLEN_CAHN, bsde.BLACK_SCHOLES])
def test_gradient_matches_central_differences(problem):
    d, w, N, T, B, x0 = 3, 5, 3, 0.5, 6, 0.7
    p = _params(problem + 3, d, w, N)
    r = nais.iteration(problem, d, w, N, T, p, 2, 1, np.arange(B), B, x0=x0)
    fd = np.zeros_like(p)
    h = 1e-6
    for i in range(p.size):
        e = np.zeros_like(p)
        e[i] = h
        fd[i] = (nais.iteration(problem, d, w, N, T, p + e, 2, 1, np.arange(B), B, x0=x0,
                                want_grad=False)["loss"]
                 - nais.iteration(problem, d, w, N, T, p - e, 2, 1, np.arange(B), B, x0=x0,
                                  want_grad=False)["loss"]) / (2 * h)
    assert np.max(np.abs(r["grad"] - fd)) <= 1e-6 * np.max(np.abs(fd))


def test_build_A_examples_and_spectrum():
    np.testing.assert_allclose(nais.build_A(np.zeros((2, 2))), -0.01 * np.eye(2))
    np.testing.assert_allclose(nais.build_A(np.eye(2)), -1.01 * np.eye(2))
    np.testing.assert_allclose(nais.build_A(np.array([[1.0, 1.0], [0.0, 0.0]])),
                               [[-1.01, -1.0], [-1.0, -1.01]])
    rng = np.random.default_rng(0)
    for _ in range(1000):
        k = rng.integers(1, 17)
        A = nais.build_A(rng.uniform(-1, 1, (k, k)))
        assert np.array_equal(A, A.T)
        assert np.linalg.eigvalsh(A).max() <= -0.01 + 1e-12


def test_project_R():
    R = np.diag([0.5 ** 0.5, 0.0])                      # ‖RᵀR‖_F = 0.5
    assert np.array_equal(nais.project_R(R), R)
    P = nais.project_R(2.0 * np.eye(2))                 # ‖RᵀR‖_F = 4√2 > 0.99
    assert abs(np.linalg.norm(P.T @ P) - 0.99) < 1e-14
    rng = np.random.default_rng(1)
    for _ in range(200):
        R = rng.uniform(-1, 1, (6, 6))
        P = nais.project_R(R)
        assert np.linalg.norm(P.T @ P) <= max(0.99, 0.0) + 1e-12
        assert np.linalg.norm(P.T @ P) <= np.linalg.norm(R.T @ R) + 1e-12
        np.testing.assert_allclose(nais.project_R(P), P, rtol=1e-13, atol=0)


@pytest.mark.parametrize("problem", [bsde.HJB, bsde.ALLEN_CAHN])
def test_zero_block_equals_residual_oracle(problem):
    """Pin N4: R = B = C = 0 makes A2 = -εH1 ≤ 0, so H2 = H1; the residual-block
    net with W2 = b2 = 0 also has H2 = H1.  Loss and the W1, b1, W3, b3, Y0
    gradients must agree with oracle/bsde.py."""
    d, w, N, T, M = 4, 6, 3, 0.5, 50
    p = _params(7, d, w, N, scale=0.1)
    _, nets = nais.unpack(p, d, w, N)
    q = np.zeros(bsde.num_params(d, w, N))
    q[0] = p[0]
    _, qnets = bsde.unpack(q, d, w, N)
    for net, qn in zip(nets, qnets):
        net["R"][...] = 0.0
        net["B"][...] = 0.0
        net["C"][...] = 0.0
        for k in ("W1", "b1", "W3", "b3"):
            qn[k][...] = net[k]
    a = nais.iteration(problem, d, w, N, T, p, 0, 3, np.arange(M), M)
    b = bsde.iteration(problem, d, w, N, T, q, 0, 3, np.arange(M), M)
    assert abs(a["loss"] - b["loss"]) <= 1e-13 * b["loss"]
    _, ga = nais.unpack(a["grad"], d, w, N)
    _, gb = bsde.unpack(b["grad"], d, w, N)
    assert abs(a["grad"][0] - b["grad"][0]) <= 1e-12 * abs(b["grad"][0])
    for x, y in zip(ga, gb):
        for k in ("W1", "b1", "W3", "b3"):
            np.testing.assert_allclose(x[k], y[k], rtol=1e-10, atol=1e-14)


def test_init_is_projected():
    d, w, N = 10, 20, 3
    p = nais.init_params(0, d, w, N)
    _, nets = nais.unpack(p, d, w, N)
    for net in nets:
        assert np.linalg.norm(net["R"].T @ net["R"]) <= 0.99 + 1e-12
        assert not net["b1"].any() and not net["C"].any() and not net["b3"].any()
        a = np.sqrt(6.0 / (w + d))
        assert np.all(np.abs(net["B"]) <= a) and np.abs(net["B"]).max() > 0.5 * a
