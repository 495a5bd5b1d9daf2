"""Pins of the oracle's rollout, loss, adjoint, Adam and prolongation.

Each test pins a part of oracle/bsde.py to something other than itself
(DESIGN.md §Pins): algebraic identities of the method, exact martingale
identities, closed forms, brute-force finite differences, and invariants.
"""
import numpy as np
import pytest
from scipy import integrate

from oracle import bsde, closed_forms as cf, philox


# ---------------------------------------------------------------- H1: heat optimum
@pytest.mark.parametrize("N", [5, 10])
def test_heat_optimum_pathwise_identity(N):
    """Pin H1: at the hand-built optimum, R = 2dT - 2 Σ_n |ΔW_n|² path-wise.
    Exercises Euler X, the Z-net (Eq. 7), the Y update and g."""
    d, T, B = 10, 1.0, 512
    p, w = cf.heat_optimum_params(d, T, N)
    r = bsde.iteration(bsde.HEAT, d, w, N, T, p, 0, 3, np.arange(B), B, want_grad=False)
    S = sum(np.sum(philox.brownian_increments(0, 3, n, np.arange(B), d, T / N) ** 2, axis=1)
            for n in range(N))
    assert np.max(np.abs(r["R"] - (2 * d * T - 2 * S))) < 1e-11


def test_heat_optimum_loss_floor():
    """E[L*] = 8dT²/N = 16 for config 1 (golden heat_floor_d10_T1_N5); sd of the
    batch mean is sqrt(573.44/B)."""
    d, T, N, B = 10, 1.0, 5, 16384
    p, w = cf.heat_optimum_params(d, T, N)
    r = bsde.iteration(bsde.HEAT, d, w, N, T, p, 0, 0, np.arange(B), B, want_grad=False)
    assert abs(r["loss"] - 16.0) < 4.0 * np.sqrt(573.44 / B)
    assert cf.heat_optimum_expected_loss(d, T, N) == 16.0


def test_heat_optimum_is_stationary():
    """Pin H2: E[∇L] = 0 at the exact optimum.  Two independent batches: for a
    mean-zero estimator |g1+g2|² ≈ |g1-g2|²; a biased adjoint breaks the ratio."""
    d, T, N, B = 4, 1.0, 3, 4096
    p, w = cf.heat_optimum_params(d, T, N)
    p = p + 0.0
    g1 = bsde.iteration(bsde.HEAT, d, w, N, T, p, 0, 0, np.arange(B), B)["grad"]
    g2 = bsde.iteration(bsde.HEAT, d, w, N, T, p, 0, 1, np.arange(B), B)["grad"]
    ratio = np.sum((g1 + g2) ** 2) / np.sum((g1 - g2) ** 2)
    assert 0.6 < ratio < 1.6, ratio
    # ... while a perturbed (non-optimal) point has a gradient far above noise
    q = p.copy()
    q[0] += 1.0
    h1 = bsde.iteration(bsde.HEAT, d, w, N, T, q, 0, 0, np.arange(B), B)["grad"]
    h2 = bsde.iteration(bsde.HEAT, d, w, N, T, q, 0, 1, np.arange(B), B)["grad"]
    assert np.sum((h1 + h2) ** 2) / np.sum((h1 - h2) ** 2) > 3.0
    assert abs(h1[0] - 2.0) < 0.2          # ∂L/∂Y0 = 2 E[R] = 2·1


# ---------------------------------------------------------------- HJB driver
def test_hjb_exponential_martingale():
    """With f = -|z|²/2 (λ = 1) and any adapted Z, exp(-(Y_N - Y0)) =
    Π_n exp(-Z_n·ΔW_n - |Z_n|²Δt/2) is a discrete exponential martingale, so
    E[exp(-(Y_N - Y0))] = 1 exactly (Gaussian ΔW).  A wrong sign or factor in
    f (R2, R10) moves the mean by a factor e^{±Σ|Z|²Δt/2}."""
    d, w, N, T, B = 4, 8, 4, 1.0, 200000
    p = bsde.init_params(11, d, w, N)
    _, nets = bsde.unpack(p, d, w, N)
    for net in nets:
        net["b3"][...] = 0.25
        net["W3"][...] *= 0.3
    r = bsde.iteration(bsde.HJB, d, w, N, T, p, 5, 0, np.arange(B), B, want_grad=False,
                       keep=True)
    qv = sum(np.sum(t[6] ** 2, axis=1) for t in r["trace"]) * (T / N)
    assert 0.3 < qv.mean() < 2.0                      # the test has power
    e = np.exp(-(r["Y_N"] - p[0]))
    assert abs(e.mean() - 1.0) < 5.0 * e.std() / np.sqrt(B)
    # the flipped driver would give a mean far from 1
    e_flip = np.exp(-(r["Y_N"] - p[0]) + qv)
    assert abs(e_flip.mean() - 1.0) > 20.0 * e_flip.std() / np.sqrt(B)


def test_hjb_zero_z_keeps_y0():
    """Pin H11: Z ≡ 0 ⇒ f(y, 0) = 0 ⇒ Y_N = Y0 and R = Y0 - g(√2 Σ ΔW)."""
    d, w, N, T, B = 6, 7, 5, 1.0, 300
    p = bsde.init_params(2, d, w, N)
    _, nets = bsde.unpack(p, d, w, N)
    for net in nets:
        net["W3"][...] = 0.0
    r = bsde.iteration(bsde.HJB, d, w, N, T, p, 0, 9, np.arange(B), B, want_grad=False)
    XN = np.sqrt(2.0) * sum(philox.brownian_increments(0, 9, n, np.arange(B), d, T / N)
                            for n in range(N))
    g = np.log(0.5 * (1.0 + np.sum(XN * XN, 1)))
    assert np.allclose(r["Y_N"], p[0], rtol=0, atol=1e-14)
    assert np.allclose(r["R"], p[0] - g, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- Allen-Cahn driver
def test_allen_cahn_zero_z_converges_to_ode():
    """With Z ≡ 0 the Y recursion is forward Euler for y' = -(y - y³)
    (f = y - y³, R12).  Its limit is the exact ODE solution
    (closed form, cross-checked with scipy's solve_ivp); the error is O(1/N)."""
    d, w, T, y0 = 3, 4, 0.3, 0.5
    exact = cf.allen_cahn_zero_z_ode(y0, T)
    sol = integrate.solve_ivp(lambda t, y: -(y - y ** 3), (0, T), [y0], rtol=1e-12, atol=1e-14)
    assert abs(sol.y[0, -1] - exact) < 1e-10
    ys = []
    for N in (20, 40, 80, 160):
        p = bsde.init_params(0, d, w, N)
        p[0] = y0
        _, nets = bsde.unpack(p, d, w, N)
        for net in nets:
            net["W3"][...] = 0.0
        r = bsde.iteration(bsde.ALLEN_CAHN, d, w, N, T, p, 0, 0, np.arange(8), 8,
                           want_grad=False)
        assert np.ptp(r["Y_N"]) == 0.0
        ys.append(r["Y_N"][0])
    errs = [y - exact for y in ys]
    for a, b in zip(errs, errs[1:]):
        assert 1.8 < a / b < 2.2                       # first order
    assert abs(2 * ys[-1] - ys[-2] - exact) < 2e-6     # Richardson
    # survey's stated value for N = 20 (Appendix A)
    assert abs(ys[0] - 0.392951276) < 1e-9


# ---------------------------------------------------------------- Black-Scholes (NEXT-3)
def test_black_scholes_zero_z_growth_and_terminal():
    """Pin BS1: Z ≡ 0 ⇒ f = -r y ⇒ Y_N = Y0 (1 + rΔt)^N exactly (closed form of the
    linear recursion), and X_N = x0 Π_n (1 + σ ΔW_n) component-wise (the Euler
    step of dX = σ diag(X) dW), so R = Y_N - ‖X_N‖² (g) is known
    from the increments alone."""
    d, w, N, T, B, x0 = 5, 6, 7, 1.0, 200, 1.3
    p = bsde.init_params(4, d, w, N)
    _, nets = bsde.unpack(p, d, w, N)
    for net in nets:
        net["W3"][...] = 0.0
    r = bsde.iteration(bsde.BLACK_SCHOLES, d, w, N, T, p, 0, 3, np.arange(B), B, x0=x0,
                       want_grad=False)
    assert np.allclose(r["Y_N"], p[0] * cf.bs_zero_z_growth(N, T), rtol=1e-13, atol=0)
    XN = np.full((B, d), x0)
    for n in range(N):
        XN = XN * (1.0 + 0.4 * philox.brownian_increments(0, 3, n, np.arange(B), d, T / N))
    assert np.allclose(r["R"], r["Y_N"] - np.sum(XN * XN, 1), rtol=1e-12, atol=1e-12)


def test_black_scholes_second_moment():
    """Pin BS2: E‖X_N‖² = d x0² (1 + σ²Δt)^N exactly for the Euler scheme (each
    step multiplies E[X_i²] by 1 + σ²Δt); checked within 4 standard errors over
    the oracle's Philox paths, and -- a wrong σ or an additive step would move
    it by > 30 SE -- against the continuous closed form's growth e^{σ²T}."""
    d, N, T, B, x0 = 8, 10, 1.0, 40000, 2.0
    X = np.full((B, d), x0)
    for n in range(N):
        X = bsde.forward_step(bsde.BLACK_SCHOLES, X, philox.brownian_increments(0, 0, n, np.arange(B), d, T / N))
    s = np.sum(X * X, 1)
    se = s.std() / np.sqrt(B)
    assert abs(s.mean() - cf.bs_discrete_second_moment(d, N, T, x0)) < 4 * se
    assert abs(cf.bs_discrete_second_moment(d, N, T, x0) - d * x0 * x0 * np.exp(0.16 * T)) < 0.02 * d * x0 * x0
    additive = d * x0 * x0 + d * 0.16 * T          # X + σΔW instead of X + σXΔW
    assert abs(s.mean() - additive) > 30 * se


def test_black_scholes_closed_form():
    """u(x, t) = e^{(r+σ²)(T-t)} ‖x‖² solves u_t = -½Tr[σ² diag(x²) D²u] + r(u - (Du)ᵀx)
    (P:293-297), checked by finite differences at random points; and the driver
    f = -r(y - Σz/σ) with z = σ x ⊙ ∇u reproduces the PDE's right-hand side term."""
    rng = np.random.default_rng(0)
    d, r, sg, T = 4, 0.05, 0.4, 1.0
    u = lambda x, t: np.exp((r + sg * sg) * (T - t)) * np.sum(x * x)
    for _ in range(5):
        x, t, h = rng.uniform(0.5, 1.5, d), rng.uniform(0, T), 1e-4
        ut = (u(x, t + h) - u(x, t - h)) / (2 * h)
        grad = np.array([(u(x + h * e, t) - u(x - h * e, t)) / (2 * h) for e in np.eye(d)])
        lap = np.array([(u(x + h * e, t) - 2 * u(x, t) + u(x - h * e, t)) / h ** 2 for e in np.eye(d)])
        rhs = -0.5 * sg * sg * np.sum(x * x * lap) + r * (u(x, t) - grad @ x)
        assert abs(ut - rhs) < 1e-5 * abs(ut)
        z = sg * x * grad
        f = bsde.driver_f(bsde.BLACK_SCHOLES, np.array(u(x, t)), z[None, :])
        assert abs(-f - r * (u(x, t) - grad @ x)) < 1e-6 * abs(f)
    assert abs(cf.bs_u0(100, 1.0) - 100 * np.exp(0.21)) < 1e-12


# ---------------------------------------------------------------- H6: FD gradients
@pytest.mark.parametrize("problem", [bsde.HEAT, bsde.HJB, bsde.ALLEN_CAHN, bsde.BLACK_SCHOLES])
@pytest.mark.parametrize("d,w,N,B", [(2, 4, 2, 4), (3, 8, 3, 8)])
def test_gradient_matches_central_differences(problem, d, w, N, B):
    T, seed, it, x0 = 0.5, 3, 1, 0.3
    p = bsde.init_params(seed, d, w, N)
    rng = np.random.default_rng(7 + d)
    p[1:] += 0.1 * rng.standard_normal(p.size - 1)     # non-zero biases
    p[0] = 0.4
    r = bsde.iteration(problem, d, w, N, T, p, seed, it, np.arange(B), B, x0=x0, keep=True)
    # no ReLU kink within reach of the FD step
    amin = min(min(np.abs(t[2]).min(), np.abs(t[4]).min()) for t in r["trace"])
    assert amin > 1e-4
    h = 1e-6
    fd = np.empty_like(p)
    for i in range(p.size):
        e = np.zeros_like(p)
        e[i] = h
        lp = bsde.iteration(problem, d, w, N, T, p + e, seed, it, np.arange(B), B, x0=x0,
                            want_grad=False)["loss"]
        lm = bsde.iteration(problem, d, w, N, T, p - e, seed, it, np.arange(B), B, x0=x0,
                            want_grad=False)["loss"]
        fd[i] = (lp - lm) / (2 * h)
    g = r["grad"]
    scale = np.abs(g).max()
    assert np.max(np.abs(g - fd)) < 1e-6 * scale + 1e-9, np.max(np.abs(g - fd)) / scale


def test_net0_is_a_trainable_z0():
    """Pin H7 / R3: with X0 = 0 and zero biases, net_0 sees A1 = A2 = 0, so only
    its b3 (= Z0, P:78 'Z0 treated as parameter') receives gradient."""
    d, w, N, T, B = 5, 6, 3, 1.0, 64
    p = bsde.init_params(0, d, w, N)
    state = bsde.AdamState(p.size)
    P = bsde.step_size(d, w)
    p_start = p.copy()
    for it in range(3):
        r = bsde.iteration(bsde.HJB, d, w, N, T, p, 0, it, np.arange(B), B)
        g = r["grad"][1:1 + P]
        assert np.all(g[:P - d] == 0.0)
        assert np.any(g[P - d:] != 0.0)
        bsde.adam_step(p, r["grad"], state, 1e-2, loss=r["loss"])
    assert np.array_equal(p[1:1 + P - d], p_start[1:1 + P - d])


def test_shard_sum_equals_full_batch():
    """§8(e): any partition of the global paths gives the same loss and gradient
    up to summation order."""
    d, w, N, T, B = 4, 6, 3, 0.3, 48
    p = bsde.init_params(1, d, w, N)
    full = bsde.iteration(bsde.ALLEN_CAHN, d, w, N, T, p, 0, 2, np.arange(B), B)
    parts = [bsde.iteration(bsde.ALLEN_CAHN, d, w, N, T, p, 0, 2, idx, B)
             for idx in np.array_split(np.arange(B), 3)]
    assert np.isclose(sum(q["loss"] for q in parts), full["loss"], rtol=1e-13)
    assert np.allclose(sum(q["grad"] for q in parts), full["grad"], rtol=1e-12, atol=1e-15)
    # permutation invariance of the loss
    perm = bsde.iteration(bsde.ALLEN_CAHN, d, w, N, T, p, 0, 2, np.arange(B)[::-1], B)
    assert np.isclose(perm["loss"], full["loss"], rtol=1e-13)


# ---------------------------------------------------------------- Adam (H8)
def test_adam_constant_gradient_moves_lr_per_step():
    """With a constant gradient g, m̂ = g and v̂ = g² exactly at every t, so every
    step moves θ by exactly lr·g/(|g|+ε); step 1 ≈ -lr·sign(g)."""
    rng = np.random.default_rng(0)
    g = rng.standard_normal(50)
    g[0] = 0.0
    th = rng.standard_normal(50)
    st = bsde.AdamState(50)
    lr = 1e-2
    for k in range(1, 6):
        before = th.copy()
        assert bsde.adam_step(th, g, st, lr)
        assert np.allclose(before - th, lr * g / (np.abs(g) + 1e-8), rtol=1e-9, atol=1e-15)
        assert st.t == k
    assert th[0] == before[0]                          # zero gradient: unchanged


def test_adam_divergence_guard_skips_update():
    th = np.ones(4)
    st = bsde.AdamState(4)
    assert not bsde.adam_step(th, np.array([1, np.nan, 0, 0.]), st, 0.1)
    assert not bsde.adam_step(th, np.ones(4), st, 0.1, loss=2e12)
    assert np.all(th == 1.0) and st.t == 0 and np.all(st.m == 0)


# ---------------------------------------------------------------- prolongation (H9)
def test_prolongate_copy_and_interp():
    d, w, N = 3, 4, 4
    p = bsde.init_params(0, d, w, N)
    P = bsde.step_size(d, w)
    c = bsde.prolongate(p, d, w, N, bsde.COPY)
    assert c.size == bsde.num_params(d, w, 2 * N) and c[0] == p[0]
    src = p[1:].reshape(N, P)
    fine = c[1:].reshape(2 * N, P)
    for k in range(2 * N):
        assert np.array_equal(fine[k], src[k // 2])
    i = bsde.prolongate(p, d, w, N, bsde.INTERP)[1:].reshape(2 * N, P)
    for n in range(N):
        assert np.array_equal(i[2 * n], src[n])
    for n in range(N - 1):
        assert np.allclose(i[2 * n + 1], 0.5 * (src[n] + src[n + 1]))
    assert np.array_equal(i[-1], src[-1])


def test_keep_adam_prolongation_commutes_with_adam():
    """R14b (keep the Adam state across a level change): Adam is elementwise, so with
    copy prolongation of the parameters *and* the moments (t kept) one Adam step on
    the fine grid, restricted to the even steps 2c, is the coarse Adam step with
    that restricted gradient.  A reset moment, a reset t (bias correction), or
    moments shifted against their parameters break it; an odd fine step 2c+1 with
    gradient g equals the coarse update with g as well."""
    d, w, N = 3, 4, 3
    P = bsde.step_size(d, w)
    rng = np.random.default_rng(5)
    p = bsde.init_params(1, d, w, N)
    st = bsde.AdamState(p.size)
    for _ in range(3):   # a non-trivial coarse state (t = 3, m, v != 0)
        assert bsde.adam_step(p, rng.normal(size=p.size), st, 1e-2)
    q = bsde.prolongate(p, d, w, N, bsde.COPY)
    sf = bsde.prolongate_adam(st, d, w, N, bsde.COPY)
    assert sf.t == st.t and sf.m.size == q.size
    g = rng.normal(size=q.size)
    assert bsde.adam_step(q, g, sf, 1e-2)
    for par in (0, 1):
        sel = np.concatenate([[0], (np.arange(2 * N * P).reshape(2 * N, P)[par::2] + 1).reshape(-1)])
        pc, sc = p.copy(), bsde.AdamState(p.size)
        sc.m, sc.v, sc.t = st.m.copy(), st.v.copy(), st.t
        assert bsde.adam_step(pc, g[sel], sc, 1e-2)
        assert np.allclose(q[sel], pc, rtol=0, atol=1e-15)
        assert np.allclose(sf.m[sel], sc.m, rtol=0, atol=1e-15)
    # against the R14 reset: the first fine step then moves every entry by ~lr
    q2, s2 = bsde.prolongate(p, d, w, N, bsde.COPY), bsde.AdamState(q.size)
    bsde.adam_step(q2, g, s2, 1e-2)
    assert not np.allclose(q2, q)
    # the interp rule moves the moments with their parameters (midpoints of both)
    si = bsde.prolongate_adam(st, d, w, N, bsde.INTERP)
    mi = si.m[1:].reshape(2 * N, P)
    src = st.m[1:].reshape(N, P)
    assert np.allclose(mi[1], 0.5 * (src[0] + src[1])) and np.array_equal(mi[-1], src[-1])


def test_keep_adam_schedule_one_level_is_single_level():
    """With one level the keep-Adam schedule is plain training (no level change)."""
    d, w, N, T, B = 3, 4, 2, 1.0, 16
    p0 = bsde.init_params(0, d, w, N)
    a, _ = bsde.train_multilevel(bsde.HJB, d, w, [N], T, p0.copy(), 0, B, [3], 1e-2, keep_adam=True)
    b, _, _ = bsde.train(bsde.HJB, d, w, N, T, p0.copy(), 0, B, 3, 1e-2)
    assert np.array_equal(a, b)


def test_prolongated_heat_optimum_stays_optimal():
    """The heat optimum is time-independent, so its prolongation is the optimum
    on the 2N grid: the path-wise identity holds there too (floor 8dT²/(2N))."""
    d, T, N, B = 10, 1.0, 5, 256
    p, w = cf.heat_optimum_params(d, T, N)
    q = bsde.prolongate(p, d, w, N, bsde.COPY)
    r = bsde.iteration(bsde.HEAT, d, w, 2 * N, T, q, 0, 0, np.arange(B), B, want_grad=False)
    S = sum(np.sum(philox.brownian_increments(0, 0, n, np.arange(B), d, T / (2 * N)) ** 2, 1)
            for n in range(2 * N))
    assert np.max(np.abs(r["R"] - (2 * d * T - 2 * S))) < 1e-11


def test_single_level_schedule_equals_single_level_training():
    """a one-level schedule is single-level training."""
    d, w, N, T, B = 3, 4, 2, 1.0, 16
    p0 = bsde.init_params(0, d, w, N)
    a, _, la = bsde.train(bsde.HJB, d, w, N, T, p0.copy(), 0, B, 4, 1e-2)
    b, hist = bsde.train_multilevel(bsde.HJB, d, w, [N], T, p0.copy(), 0, B, [4], 1e-2)
    assert np.array_equal(a, b) and [h[2] for h in hist] == la


# ---------------------------------------------------------------- init (R7) and bf16 (R17)
def test_init_ranges():
    d, w, N = 100, 110, 2
    p = bsde.init_params(0, d, w, N)
    y0, nets = bsde.unpack(p, d, w, N)
    assert 0 < y0[0] < 1
    for net in nets:
        for name, (fo, fi) in (("W1", (w, d)), ("W2", (w, w)), ("W3", (d, w))):
            a = np.sqrt(6.0 / (fi + fo))
            assert np.abs(net[name]).max() <= a
            assert abs(net[name].std() - a / np.sqrt(3)) < 0.05 * a
        for b in ("b1", "b2", "b3"):
            assert np.all(net[b] == 0)
    assert not np.array_equal(nets[0]["W1"], nets[1]["W1"])


def test_round_bf16_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).standard_normal(10000) * 10.0 ** np.random.default_rng(1).integers(-5, 5, 10000)
    ref = torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(bsde.round_bf16(x), ref)


def test_round_fp16_matches_torch():
    """The binary16 rounding of ΔW_n in the tensor-core reading of R17: RNE as
    torch's conversion, over normal and subnormal half-precision magnitudes."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    x = rng.standard_normal(20000) * 10.0 ** rng.integers(-7, 4, 20000)
    ref = torch.tensor(x, dtype=torch.float32).to(torch.float16).to(torch.float64).numpy()
    assert np.array_equal(bsde.round_fp16(x), ref)


@pytest.mark.parametrize("problem", [bsde.HEAT, bsde.HJB, bsde.ALLEN_CAHN, bsde.BLACK_SCHOLES])
def test_tc_emulation_with_identity_roundings_is_the_exact_oracle(problem):
    """Structural pin of the tensor-core rounding model (iteration(tc=True)): with
    the roundings replaced by the identity, the folded biases, the bf16-formed
    residual sum, the ΔW_n storage and the adjoint's operand sites collapse to
    the exact algebra, bit for bit (so the model differs from the oracle only
    where it rounds), and with the roundings in place it does round."""
    d, w, N, T, B = 7, 9, 3, 1.0, 40
    p = bsde.init_params(2, d, w, N)
    p[1:] += 0.05 * np.random.default_rng(1).standard_normal(p.size - 1)
    x0 = 0.7 if problem == bsde.BLACK_SCHOLES else 0.0
    ex = bsde.iteration(problem, d, w, N, T, p, 0, 1, np.arange(B), B, x0=x0, kink_band=1e-3)
    idn = bsde.iteration(problem, d, w, N, T, p, 0, 1, np.arange(B), B, x0=x0, kink_band=1e-3,
                         tc=True, rb=bsde._ident, rh=bsde._ident)
    assert idn["loss"] == ex["loss"]
    assert np.array_equal(idn["grad"], ex["grad"]) and np.array_equal(idn["slack"], ex["slack"])
    tc = bsde.iteration(problem, d, w, N, T, p, 0, 1, np.arange(B), B, x0=x0, tc=True)
    assert tc["loss"] != ex["loss"] and not np.array_equal(tc["grad"], ex["grad"])
    # within the bf16 error model: operands carry 2^-9 relative rounding
    assert abs(tc["loss"] - ex["loss"]) <= 2e-2 * ex["loss"]
    assert np.linalg.norm(tc["grad"] - ex["grad"]) <= 2e-2 * np.linalg.norm(ex["grad"])


def test_tc_emulation_rounds_at_each_documented_site():
    """Each rounding site of the model moves the result on its own (a site the
    model forgot would leave the result unchanged when only it is switched):
    only ΔW_n in binary16, and only the bf16 operand rounding."""
    d, w, N, T, B = 10, 12, 3, 1.0, 64
    p = bsde.init_params(3, d, w, N)
    p[1:] += 0.05 * np.random.default_rng(2).standard_normal(p.size - 1)
    ex = bsde.iteration(bsde.HJB, d, w, N, T, p, 0, 0, np.arange(B), B)
    only_h = bsde.iteration(bsde.HJB, d, w, N, T, p, 0, 0, np.arange(B), B, tc=True,
                            rb=bsde._ident)
    only_b = bsde.iteration(bsde.HJB, d, w, N, T, p, 0, 0, np.arange(B), B, tc=True,
                            rh=bsde._ident)
    for r, lo, hi in ((only_h, 1e-7, 3e-3), (only_b, 1e-6, 2e-2)):
        rel = np.linalg.norm(r["grad"] - ex["grad"]) / np.linalg.norm(ex["grad"])
        assert lo < rel < hi, rel
    # binary16 ΔW: the Y update sees Σ Z·fp16(ΔW); X advances with the exact ΔW
    assert np.array_equal(only_h["X_N"], ex["X_N"])


def test_zero_head_init_keeps_allen_cahn_bounded():
    """R7b: with a Xavier head the Allen-Cahn rollout explodes at config-3 sizes
    (Y leaves [-1, 1] and the cubic driver diverges); with W3 = 0 (Z ≡ 0) Y_n
    follows the bounded scalar ODE map."""
    d, w, N, T, B = 100, 110, 20, 0.3, 256
    with np.errstate(all="ignore"):
        bad = bsde.iteration(bsde.ALLEN_CAHN, d, w, N, T, bsde.init_params(0, d, w, N), 0, 0,
                             np.arange(B), B, want_grad=False)
    assert not np.isfinite(bad["loss"]) or bad["loss"] > 1e6
    p = bsde.init_params(0, d, w, N, zero_head=True)
    _, nets = bsde.unpack(p, d, w, N)
    assert all(not net["W3"].any() for net in nets) and nets[1]["W1"].any()
    r = bsde.iteration(bsde.ALLEN_CAHN, d, w, N, T, p, 0, 0, np.arange(B), B)
    assert np.isfinite(r["loss"]) and r["loss"] < 1.0 and np.all(np.isfinite(r["grad"]))


def test_kink_slack_bounds_mask_flips():
    """The slack returned with kink_band bounds the gradient change when every
    pre-activation inside the band flips its ReLU mask (emulated by evaluating
    the backward masks as 1[A > shift])."""
    d, w, N, T, B = 6, 10, 3, 1.0, 64
    p = bsde.init_params(4, d, w, N)
    p[1:] += 0.05 * np.random.default_rng(0).standard_normal(p.size - 1)
    for problem in (bsde.HJB, bsde.ALLEN_CAHN):
        base = bsde.iteration(problem, d, w, N, T, p, 0, 0, np.arange(B), B, kink_band=0.05,
                              keep=True)
        shifted = bsde.iteration(problem, d, w, N, T, p, 0, 0, np.arange(B), B, mask_shift=0.002)
        flipped = sum(int(np.sum((A > 0) & (A <= 0.002))) for t in base["trace"]
                      for A in (t[2], t[4]))
        assert flipped > 0
        diff = np.abs(shifted["grad"] - base["grad"])
        assert diff.max() > 0                           # the flips did change the gradient
        assert np.all(diff <= base["slack"] * 1.05 + 1e-12)


# ------------------------------------------------- coupled multilevel paths (NEXT-3)
def test_coupled_increments_share_the_brownian_path():
    """Pin C1 (SPEC S:314-322 coarsen_increments): the coupled increments of every
    level sum to the same W_T as the finest grid's own increments (the levels
    simulate one underlying path), factor 1 is the plain generator, and a coarse
    increment has variance Δt_coarse with no correlation between steps."""
    d, T, Nf, seed, it = 4, 1.0, 80, 7, 3
    m = np.arange(2000)
    WT = sum(philox.brownian_increments(seed, it, k, m, d, T / Nf) for k in range(Nf))
    for N in (5, 10, 20, 40, 80):
        f = Nf // N
        inc = [philox.coupled_increments(seed, it, n, m, d, T / N, f) for n in range(N)]
        assert np.max(np.abs(sum(inc) - WT)) < 1e-12
    np.testing.assert_array_equal(philox.coupled_increments(seed, it, 3, m, d, 0.05, 1),
                                  philox.brownian_increments(seed, it, 3, m, d, 0.05))
    big = np.arange(50000)
    a = philox.coupled_increments(seed, it, 0, big, 2, 0.2, 16).ravel()
    b = philox.coupled_increments(seed, it, 1, big, 2, 0.2, 16).ravel()
    assert abs(a.var() / 0.2 - 1.0) < 0.02
    assert abs(np.mean(a * b)) / 0.2 < 0.02
    with pytest.raises(ValueError):
        philox.coupled_increments(seed, it, 0, m, d, 0.1, 0)


def test_coupled_levels_share_terminal_state():
    """Pin C2: heat with Z ≡ 0 (zero head, zero biases) has Y_N = Y0 and X_N = √2 W_T,
    so with coupled paths every level's residuals equal the finest grid's exactly."""
    d, w, T, B, Nf = 6, 8, 1.0, 64, 16
    ref = None
    for N in (2, 4, 8, 16):
        p = bsde.init_params(1, d, w, N, zero_head=True)
        r = bsde.iteration(bsde.HEAT, d, w, N, T, p, 5, 2, np.arange(B), B, want_grad=False,
                           coupled_factor=Nf // N)
        ref = r["R"] if ref is None else ref
        assert np.max(np.abs(r["R"] - ref)) < 1e-12


def test_coupled_gbm_strong_order_half():
    """Pin C3 (SPEC invariant "strong convergence order ½", fig:multilevel): the
    Black-Scholes Euler step on coupled levels against the exact geometric Brownian
    motion x0·exp(-σ²T/2 + σW_T) of the shared path: the RMS terminal error shrinks by
    ≈ √2 per halving of Δt (successive ratios in [1.2, 1.7])."""
    d, T, x0, B, Nf = 1, 1.0, 1.0, 4096, 64
    m = np.arange(B)
    WT = sum(philox.brownian_increments(0, 0, k, m, d, T / Nf) for k in range(Nf))
    exact = x0 * np.exp(-0.5 * bsde.BS_SIGMA ** 2 * T + bsde.BS_SIGMA * WT)
    errs = []
    for N in (8, 16, 32, 64):
        X = np.full((B, d), x0)
        for n in range(N):
            X = bsde.forward_step(bsde.BLACK_SCHOLES, X,
                                  philox.coupled_increments(0, 0, n, m, d, T / N, Nf // N))
        errs.append(np.sqrt(np.mean((X - exact) ** 2)))
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(1.2 <= r <= 1.7 for r in ratios), ratios
