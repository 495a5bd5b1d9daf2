"""Closed forms the oracle is pinned against (TEST INFRASTRUCTURE ONLY).

heat       u(0,x0) = |x0|² + 2dT (BASELINE.json config 1; R13) and a hand-built
           exact optimum of the per-step ReLU net for it (DESIGN.md pin H1).
hjb        Cole-Hopf: u(0,x) = -ln E[exp(-g(x + √2 W_T))]  (subscript read
           as W_{T-t}, R11).  At x = 0, |√2 W_T|² = 2T χ²_d, so
           u(0,0) = -ln E[2 / (1 + 2T χ²_d)]: a 1-D quadrature.
allen_cahn linearisation u0 ≈ e^T E[g(X_T)] (R12 constants) and the Z ≡ 0 ODE
           y' = -(y - y³) whose exact solution is y(t) = (1 + (y0^-2 - 1) e^{2t})^{-1/2}.
"""
import numpy as np
from scipy import integrate, stats


def heat_u0(d, T, x0=0.0):
    return float(d * x0 * x0 + 2.0 * d * T)


def heat_optimum_params(d, T, N):
    """Exact optimum for f=0, g=|x|², σ=√2 with width w = 2d (pin H1):
    W1 = [I; -I], b1 = 0, W2 = 0, b2 = 0, W3 = 2√2 [I, -I], b3 = 0, Y0 = 2dT,
    so Z_n = 2√2 X_n = σᵀ∇u(t, X_n) and R = 2dT - 2 Σ_n |ΔW_n|² path-wise."""
    from .bsde import num_params, unpack
    w = 2 * d
    p = np.zeros(num_params(d, w, N))
    y0, nets = unpack(p, d, w, N)
    y0[0] = 2.0 * d * T
    eye = np.eye(d)
    for net in nets:
        net["W1"][...] = np.vstack([eye, -eye])
        net["W3"][...] = 2.0 * np.sqrt(2.0) * np.hstack([eye, -eye])
    return p, w


def heat_optimum_expected_loss(d, T, N):
    """E[(2dT - 2Σ|ΔW|²)²] = 4 Var(Σ|ΔW|²) = 4·N·d·2Δt² = 8dT²/N."""
    return 8.0 * d * T * T / N


def hjb_u0_quadrature(d, T, lam=1.0):
    """-(1/λ) ln E[exp(-λ g(√2 W_T))] with g = ln(0.5(1+|x|²)); λ=1 (R10, R11)."""
    assert lam == 1.0
    pdf = stats.chi2(d).pdf
    val, _ = integrate.quad(lambda r: 2.0 / (1.0 + 2.0 * T * r) * pdf(r), 0.0, np.inf,
                            limit=400, epsabs=0.0, epsrel=1e-13)
    return float(-np.log(val))


def hjb_u0_mc(d, T, K, rng):
    """Monte Carlo of the Cole-Hopf expectation with an independent numpy generator."""
    W = rng.standard_normal((K, d)) * np.sqrt(T)
    x = np.sqrt(2.0) * W
    e = 2.0 / (1.0 + np.sum(x * x, axis=1))
    return float(-np.log(e.mean())), float(e.std() / (e.mean() * np.sqrt(K)))


def expected_g_chi2(problem_g, d, T):
    """E[g(X_T)] for X_T = √2 W_T, X0 = 0, with g a function of s = |x|² = 2T χ²_d."""
    pdf = stats.chi2(d).pdf
    val, _ = integrate.quad(lambda r: problem_g(2.0 * T * r) * pdf(r), 0.0, np.inf,
                            limit=400, epsabs=0.0, epsrel=1e-13)
    return float(val)


def allen_cahn_linearised_u0(d, T):
    """Linearising f = y - y³ around 0: u0 ≈ e^T E[g(X_T)]  (survey pin H5)."""
    return float(np.exp(T) * expected_g_chi2(lambda s: 1.0 / (2.0 + 0.4 * s), d, T))


def allen_cahn_zero_z_ode(y0, T):
    """Exact solution of y' = -(y - y³), y(0) = y0, at time T (the Z ≡ 0 limit)."""
    return float((1.0 + (y0 ** -2 - 1.0) * np.exp(2.0 * T)) ** -0.5)


# ----------------------------------------------------------------------------
# Black-Scholes: dX = σ diag(X) dW, g = ‖x‖²
# ----------------------------------------------------------------------------
def bs_u0(d, T, x0=1.0, r=0.05, sigma=0.4):
    """u(x0, 0) = e^{(r+σ²)T} ‖x0‖² with x0 = x0·1."""
    return float(np.exp((r + sigma * sigma) * T) * d * x0 * x0)


def bs_discrete_second_moment(d, N, T, x0=1.0, sigma=0.4):
    """E‖X_N‖² of the Euler scheme X_{n+1,i} = X_{n,i}(1 + σΔW_{n,i}): every step
    multiplies E[X_i²] by E[(1 + σΔW)²] = 1 + σ²Δt, exactly."""
    return float(d * x0 * x0 * (1.0 + sigma * sigma * T / N) ** N)


def bs_zero_z_growth(N, T, r=0.05):
    """With Z ≡ 0 the Y recursion Y_{n+1} = Y_n - f Δt, f = -r(y - Σz/σ), is
    Y_{n+1} = (1 + rΔt) Y_n: Y_N = Y0 (1 + rΔt)^N exactly."""
    return float((1.0 + r * T / N) ** N)
