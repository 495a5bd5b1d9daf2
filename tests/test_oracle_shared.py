"""Pins of the shared-network oracle (oracle/shared.py).

Each pin fixes part of the oracle against something other than itself: central
finite differences (the reverse-over-reverse gradient and ∇ₓu), constant-network
special cases whose residuals and loss have closed forms, the residual-block
identity, and shard additivity (S1-S6).
"""
import numpy as np
import pytest

from oracle import bsde, philox, shared

PROBLEMS = [bsde.HEAT, bsde.HJB, bsde.ALLEN_CAHN, bsde.BLACK_SCHOLES]


def _params(seed, d, w, L, scale=0.3, arch=shared.FC):
    p = shared.init_params(seed, d, w, L, arch)
    rng = np.random.default_rng(seed)
    return p + scale * rng.standard_normal(p.size)      # non-zero biases, generic weights


@pytest.mark.parametrize("arch", [shared.FC, shared.RESNET, shared.NAIS])
@pytest.mark.parametrize("problem", PROBLEMS)
def test_gradient_matches_central_differences(problem, arch):
    """Pin S1: ∂L/∂Θ through ∇ₓu (reverse-over-reverse) = central differences,
    h = 1e-6, to 1e-6 of the largest component, every parameter (NAIS-Net: incl.
    R̄ = -R(Ā + Āᵀ) and the input-injection B_k, R26)."""
    d, w, L, N, T, M, x0 = 3, 5, 3, 3, 0.5, 4, 0.6
    p = _params(problem + 10 * arch, d, w, L, arch=arch)
    r = shared.iteration(problem, d, w, L, arch, N, T, p, 1, 2, np.arange(M), M, x0=x0)
    g = r["grad"]
    fd = np.zeros_like(p)
    h = 1e-6
    for i in range(p.size):
        e = np.zeros_like(p)
        e[i] = h
        lp = shared.iteration(problem, d, w, L, arch, N, T, p + e, 1, 2, np.arange(M), M, x0=x0,
                              want_grad=False)["loss"]
        lm = shared.iteration(problem, d, w, L, arch, N, T, p - e, 1, 2, np.arange(M), M, x0=x0,
                              want_grad=False)["loss"]
        fd[i] = (lp - lm) / (2 * h)
    assert np.max(np.abs(g - fd)) <= 1e-6 * np.max(np.abs(fd)), np.max(np.abs(g - fd))


@pytest.mark.parametrize("arch", [shared.FC, shared.RESNET, shared.NAIS])
def test_input_gradient_matches_central_differences(arch):
    """Pin S2: g_0 = ∇_{(t,x)} u from the reverse pass = central differences
    (NAIS-Net: through every block's input injection B_k u)."""
    d, w, L = 4, 6, 4
    p = _params(7, d, w, L, arch=arch)
    rng = np.random.default_rng(3)
    t = rng.random(5)
    X = rng.standard_normal((5, d))
    _, cache = shared.forward(p, d, w, L, arch, t, X)
    g, _ = shared.input_gradient(p, d, w, L, arch, cache)
    h = 1e-6
    for i in range(d + 1):
        tp, tm, Xp, Xm = t.copy(), t.copy(), X.copy(), X.copy()
        if i == 0:
            tp += h
            tm -= h
        else:
            Xp[:, i - 1] += h
            Xm[:, i - 1] -= h
        fd = (shared.forward(p, d, w, L, arch, tp, Xp)[0]
              - shared.forward(p, d, w, L, arch, tm, Xm)[0]) / (2 * h)
        assert np.max(np.abs(g[0][:, i] - fd)) < 1e-8


def _constant_net(d, w, L, beta):
    p = np.zeros(shared.num_params(d, w, L))
    p[-1] = beta
    return p


def test_constant_network_heat_residuals_and_loss():
    """Pin S3: u ≡ β (zero weights) has Z = 0, so for heat r_n = 0 (n < N) and
    r_N = β - |X_N|² with X_N = √2 W_T; E[L] = (β - 2dT)² + 8dT² (|X_N|² = 2T χ²_d)."""
    d, w, L, N, T, beta = 5, 4, 2, 4, 0.7, 3.0
    p = _constant_net(d, w, L, beta)
    M = 40000
    r = shared.iteration(bsde.HEAT, d, w, L, shared.FC, N, T, p, 0, 1, np.arange(M), M,
                         want_grad=False)
    assert np.all(r["r"][:N] == 0.0)
    WT = sum(philox.brownian_increments(0, 1, n, np.arange(M), d, T / N) for n in range(N))
    assert np.max(np.abs(r["r"][N] - (beta - 2.0 * np.sum(WT * WT, axis=1)))) < 1e-12
    mean = (beta - 2 * d * T) ** 2 + 8 * d * T * T
    # sd of (β - S)² with S = 2Tχ²_d, by its moments
    S = 2 * np.sum(WT * WT, axis=1)
    se = np.std((beta - S) ** 2) / np.sqrt(M)
    assert abs(r["loss"] - mean) < 4 * se


@pytest.mark.parametrize("problem", [bsde.HJB, bsde.ALLEN_CAHN, bsde.BLACK_SCHOLES])
def test_constant_network_driver_residuals(problem):
    """Pin S4: u ≡ β gives r_n = f(β, 0) Δt for n < N: HJB 0, Allen-Cahn
    (β - β³)Δt, Black-Scholes -rβΔt (the sign and scale of the driver term)."""
    d, w, L, N, T, beta = 3, 4, 2, 5, 1.0, 0.8
    p = _constant_net(d, w, L, beta)
    r = shared.iteration(problem, d, w, L, shared.FC, N, T, p, 0, 0, np.arange(7), 7, x0=1.0,
                         want_grad=False)["r"]
    expect = {bsde.HJB: 0.0, bsde.ALLEN_CAHN: (beta - beta ** 3) * T / N,
              bsde.BLACK_SCHOLES: -0.05 * beta * T / N}[problem]
    assert np.max(np.abs(r[:N] - expect)) < 1e-15


def test_resnet_zero_blocks_is_the_lift():
    """Pin S5: with zero residual blocks (W_k = 0, b_k = 0 for k ≥ 2) the ResNet
    hidden state stays the lifted input, so u equals the one-layer network's."""
    d, w, L = 4, 6, 4
    p = _params(2, d, w, L)
    layers, v, c = shared.unpack(p, d, w, L)
    for W, b in layers[1:]:
        W[...] = 0.0
        b[...] = 0.0
    q = np.concatenate([p[:w * (d + 1) + w], v, c])
    t = np.linspace(0, 1, 9)
    X = np.random.default_rng(0).standard_normal((9, d))
    a = shared.forward(p, d, w, L, shared.RESNET, t, X)[0]
    b1 = shared.forward(q, d, w, 1, shared.FC, t, X)[0]
    np.testing.assert_array_equal(a, b1)


def test_shards_sum_to_full_batch():
    """Pin S6: loss sums and gradients are additive over path shards (R5, §8(e))."""
    d, w, L, N, T, B = 3, 5, 2, 3, 1.0, 10
    p = _params(4, d, w, L)
    full = shared.iteration(bsde.HJB, d, w, L, shared.FC, N, T, p, 0, 3, np.arange(B), B)
    parts = [shared.iteration(bsde.HJB, d, w, L, shared.FC, N, T, p, 0, 3, idx, B)
             for idx in (np.arange(0, 4), np.arange(4, B))]
    assert abs(sum(q["loss"] for q in parts) - full["loss"]) < 1e-12 * full["loss"]
    assert np.max(np.abs(sum(q["grad"] for q in parts) - full["grad"])) < 1e-12 * np.max(
        np.abs(full["grad"]))


def test_init_ranges():
    d, w, L = 10, 16, 4
    p = shared.init_params(0, d, w, L)
    layers, v, c = shared.unpack(p, d, w, L)
    for k, (W, b) in enumerate(layers):
        a = np.sqrt(6.0 / (W.shape[0] + W.shape[1]))
        assert np.all(np.abs(W) <= a) and np.abs(W).max() > 0.8 * a and not b.any()
    assert np.all(np.abs(v) <= np.sqrt(6.0 / (w + 1))) and 0.0 < c[0] < 1.0


def test_nais_init_projected_and_zero_block_map():
    """NAIS-Net (R26): initial R_k satisfy ‖RᵀR‖_F ≤ 1 - ε; with R = B = C = 0 a
    block maps y to y + tanh(-εy) (SPEC nets example), so a point with h_1 = 0
    (zero lift) stays 0 through every block and u = c."""
    d, w, L = 5, 8, 3
    p = shared.init_params(1, d, w, L, shared.NAIS)
    layers, v, c = shared.unpack(p, d, w, L, shared.NAIS)
    for R, C, Bk in layers[1:]:
        assert np.linalg.norm(R.T @ R) <= 0.99 + 1e-12
        assert not C.any() and np.abs(Bk).max() > 0
    q = p.copy()
    layers, v, c = shared.unpack(q, d, w, L, shared.NAIS)
    layers[0][0][...] = 0.0
    for R, C, Bk in layers[1:]:
        R[...] = 0.0
        Bk[...] = 0.0
    u, _ = shared.forward(q, d, w, L, shared.NAIS, np.zeros(3), np.ones((3, d)))
    np.testing.assert_array_equal(u, np.full(3, c[0]))


@pytest.mark.parametrize("problem", PROBLEMS)
def test_zN_term_gradient_and_grad_g(problem):
    """R27 (P:79 optional term |Z_N - g'(X_N)|²): ∇g = central differences of g,
    and the loss gradient with the term = central differences."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((6, 3))
    h = 1e-6
    for i in range(3):
        e = np.zeros(3)
        e[i] = h
        fd = (bsde.terminal_g(problem, X + e) - bsde.terminal_g(problem, X - e)) / (2 * h)
        assert np.max(np.abs(shared.grad_g(problem, X)[:, i] - fd)) < 1e-8
    d, w, L, N, T, M, x0 = 3, 5, 2, 3, 0.5, 4, 0.6
    p = _params(problem + 40, d, w, L)
    r = shared.iteration(problem, d, w, L, shared.FC, N, T, p, 1, 2, np.arange(M), M, x0=x0, zN=True)
    r0 = shared.iteration(problem, d, w, L, shared.FC, N, T, p, 1, 2, np.arange(M), M, x0=x0)
    assert r["loss"] > r0["loss"]
    fd = np.zeros_like(p)
    for k in range(p.size):
        e = np.zeros_like(p)
        e[k] = h
        fd[k] = (shared.iteration(problem, d, w, L, shared.FC, N, T, p + e, 1, 2, np.arange(M), M,
                                  x0=x0, want_grad=False, zN=True)["loss"]
                 - shared.iteration(problem, d, w, L, shared.FC, N, T, p - e, 1, 2, np.arange(M), M,
                                    x0=x0, want_grad=False, zN=True)["loss"]) / (2 * h)
    assert np.max(np.abs(r["grad"] - fd)) <= 1e-6 * np.max(np.abs(fd))
