"""Per-step Z-networks with the NAIS-Net block, float64 (TEST INFRASTRUCTURE ONLY;
SURVEY §8(f) NEXT-2).

The per-step scheme of oracle/bsde.py with the residual block of Eq. 7
replaced by the paper's stable block ("constraining the network as
follows"):

  x(k+1) = x(k) + h σ(A x(k) + B u + C),    A = -RᵀR - εI,   ε = 0.01,  h = 1

applied to the per-step net (R25): A1 = W1 X + b1, H1 = ReLU(A1),
A2 = A H1 + B X + C (the input u of the network is X_n), H2 = H1 + h ReLU(A2),
Z = W3 H2 + b3.  After every Adam step each R_n is projected onto
‖RᵀR‖_F ≤ 1 - ε ("An additional constraint is proposed on the Frobenius
norm ‖RᵀR‖_F"; the bound follows SPEC nets.project_R, R25).

Flat layout per step: [W1 (w×d) b1 (w) R (w×w) C (w) W3 (d×w) b3 (d) B (w×d)]
after Y0 — the per-step layout of bsde.py with B appended.
"""
import numpy as np

from . import philox
from .bsde import driver_df_dy, driver_df_dz, driver_f, forward_step, terminal_g

EPS = 0.01
H_STEP = 1.0
B_TENSOR_BASE = 0x100000      # init-stream tensor ids of B_n (R25)


def step_size(d, w):
    return 2 * d * w + w * w + 2 * w + d + w * d


def num_params(d, w, N):
    return 1 + N * step_size(d, w)


def unpack(params, d, w, N):
    params = np.asarray(params)
    assert params.shape == (num_params(d, w, N),), (params.shape, num_params(d, w, N))
    nets, off = [], 1
    for _ in range(N):
        net = {}
        for name, shape in (("W1", (w, d)), ("b1", (w,)), ("R", (w, w)), ("C", (w,)),
                            ("W3", (d, w)), ("b3", (d,)), ("B", (w, d))):
            size = int(np.prod(shape))
            net[name] = params[off:off + size].reshape(shape)
            off += size
        nets.append(net)
    return params[0:1], nets


def build_A(R, eps=EPS):
    """A = -RᵀR - εI: symmetric with every eigenvalue ≤ -ε."""
    return -R.T @ R - eps * np.eye(R.shape[1])


def project_R(R, eps=EPS):
    """R unchanged if ‖RᵀR‖_F ≤ 1 - ε, else scaled by ((1-ε)/‖RᵀR‖_F)^½ so that the
    result has ‖RᵀR‖_F = 1 - ε (SPEC nets.project_R)."""
    f = np.linalg.norm(R.T @ R)
    return R if f <= 1.0 - eps else R * np.sqrt((1.0 - eps) / f)


def project(params, d, w, N):
    """Apply project_R to every step's R in place (after each optimizer step)."""
    _, nets = unpack(params, d, w, N)
    for net in nets:
        net["R"][...] = project_R(net["R"])
    return params


def init_params(seed, d, w, N, zero_head=False):
    """R7 with the NAIS-Net parameters (R25): Xavier-uniform W1, R, W3 (tensor ids
    1 + 3n + k as bsde.init_params), B_n Xavier-uniform with tensor id
    0x100000 + n, zero biases, Y0 ~ U(0,1); then every R projected."""
    p = np.zeros(num_params(d, w, N))
    y0, nets = unpack(p, d, w, N)
    y0[0] = philox.init_uniforms(seed, 0, 1)[0]
    for n, net in enumerate(nets):
        names = [("W1", 1 + 3 * n), ("R", 2 + 3 * n), ("B", B_TENSOR_BASE + n)]
        if not zero_head:
            names.append(("W3", 3 + 3 * n))
        for name, tid in names:
            fan_out, fan_in = net[name].shape
            a = np.sqrt(6.0 / (fan_in + fan_out))
            u = philox.init_uniforms(seed, tid, net[name].size)
            net[name][...] = (a * (2.0 * u - 1.0)).reshape(net[name].shape)
    return project(p, d, w, N)


def net_forward(net, X):
    A1 = X @ net["W1"].T + net["b1"]
    H1 = np.maximum(A1, 0.0)
    A = build_A(net["R"])
    A2 = H1 @ A + X @ net["B"].T + net["C"]         # A symmetric: H1 Aᵀ = H1 A
    H2 = H1 + H_STEP * np.maximum(A2, 0.0)
    Z = H2 @ net["W3"].T + net["b3"]
    return A1, H1, A, A2, H2, Z


def iteration(problem, d, w, N, T, params, seed, it, paths, batch_global, x0=0.0, lam=1.0,
              want_grad=True, kink_band=0.0, coupled_factor=1):
    """As bsde.iteration (terminal loss, hand adjoint, R19 kink slack) with the
    NAIS-Net block.  Gradient of A = -RᵀR - εI: R̄ = -R(Ā + Āᵀ)."""
    paths = np.asarray(paths, dtype=np.int64)
    B = float(batch_global)
    dt = T / N
    y0, nets = unpack(params, d, w, N)
    M = len(paths)
    X = np.full((M, d), float(x0))
    Y = np.full(M, y0[0])
    trace = []
    for n in range(N):
        dW = (philox.brownian_increments(seed, it, n, paths, d, dt) if coupled_factor == 1
              else philox.coupled_increments(seed, it, n, paths, d, dt, coupled_factor))
        A1, H1, A, A2, H2, Z = net_forward(nets[n], X)
        trace.append((X, dW, A1, H1, A, A2, H2, Z, Y))
        Y = Y - driver_f(problem, Y, Z, lam) * dt + np.sum(Z * dW, axis=-1)
        X = forward_step(problem, X, dW)
    R = Y - terminal_g(problem, X)
    out = dict(loss_sum=float(np.sum(R * R)), loss=float(np.sum(R * R) / B), R=R)
    if not want_grad:
        return out
    grad = np.zeros_like(np.asarray(params, dtype=np.float64))
    gy0, gnets = unpack(grad, d, w, N)
    slack = np.zeros_like(grad)
    _, snets = unpack(slack, d, w, N)
    abar = 2.0 * R / B
    for n in range(N - 1, -1, -1):
        X, dW, A1, H1, A, A2, H2, Z, Yn = trace[n]
        net, g = nets[n], gnets[n]
        dZ = abar[:, None] * (dW - dt * driver_df_dz(problem, Yn, Z, lam))
        g["W3"][...] = dZ.T @ H2
        g["b3"][...] = dZ.sum(0)
        dH2 = dZ @ net["W3"]
        m2 = A2 > 0.0
        dA2 = H_STEP * dH2 * m2
        gA = dA2.T @ H1
        g["R"][...] = -net["R"] @ (gA + gA.T)
        g["C"][...] = dA2.sum(0)
        g["B"][...] = dA2.T @ X
        dH1 = dH2 + dA2 @ A
        m1 = A1 > 0.0
        dA1 = dH1 * m1
        g["W1"][...] = dA1.T @ X
        g["b1"][...] = dA1.sum(0)
        if kink_band > 0.0:
            s = snets[n]
            absR = np.abs(net["R"])
            absA = np.abs(A)
            amb1 = np.abs(A1) <= kink_band * (np.abs(X) @ np.abs(net["W1"]).T + np.abs(net["b1"]))
            amb2 = np.abs(A2) <= kink_band * (np.abs(H1) @ absA + np.abs(X) @ np.abs(net["B"]).T
                                              + np.abs(net["C"]))
            e2 = H_STEP * np.abs(dH2) * amb2
            e1 = np.abs(dH1) * amb1 + (e2 @ absA) * (m1 | amb1)
            sA = e2.T @ np.abs(H1)
            s["R"][...] = absR @ (sA + sA.T)
            s["C"][...] = e2.sum(0)
            s["B"][...] = e2.T @ np.abs(X)
            s["W1"][...] = e1.T @ np.abs(X)
            s["b1"][...] = e1.sum(0)
        abar = abar * (1.0 - dt * driver_df_dy(problem, Yn, Z, lam))
    gy0[0] = abar.sum()
    out["grad"] = grad
    out["slack"] = slack
    return out


def prolongate(params, d, w, N, copy=True):
    """N -> 2N over whole step blocks (R14): copy, or the midpoint rule."""
    P = step_size(d, w)
    src = np.asarray(params)[1:].reshape(N, P)
    dst = np.empty((2 * N, P))
    dst[0::2] = src
    if copy:
        dst[1::2] = src
    else:
        dst[1:-1:2] = 0.5 * (src[:-1] + src[1:])
        dst[-1] = src[-1]
    return np.concatenate([np.asarray(params)[:1], dst.reshape(-1)])
