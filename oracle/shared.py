"""The paper's own formulation, float64 (TEST INFRASTRUCTURE ONLY).

One network u(t, x; Θ) shared by every time step (fig:neural: "we use
the same parameters for all time points"), Y_n = u(t_n, X_n), Z_n from ∇ₓu by
differentiation ("compute ∇u using automatic differentiation"), and the
residual-sum loss of Eq. 6:

  ΔW_n ~ N(0, Δt)                                Eq. 5, P:64   (philox.py, R8)
  X_{n+1} = X_n + σ(X_n) ΔW_n                    Eq. 5, P:65   (bsde.forward_step)
  Y_n = u(t_n, X_n),  z_n = σ(X_n)ᵀ ∇ₓu(t_n, X_n)  P:68-69; R2, R23
  r_n = Y_{n+1} - Y_n + f(Y_n, z_n) Δt - z_n·ΔW_n   (n < N)   Eq. 6 first term, φ = -f (R2)
  r_N = Y_N - g(X_N)                                         Eq. 6 second term
  L = (1/M) Σ_m (Σ_{n<N} r_n² + r_N²)                        Eq. 6, mean over paths (R24)

Network (R23; "4 fully connected layers and 256 neurons", P:217-220 for
the residual form): input h_0 = (t, x) ∈ R^{d+1}; for k = 1..L
  a_k = W_k h_{k-1} + b_k,   s_k = tanh(a_k),
  h_k = s_k  (FC)   or   h_k = h_{k-1} + s_k for k ≥ 2  (ResNet, h = 1)
and u = v·h_L + c.  NAIS-Net (R26): layer 1 as FC, blocks k ≥ 2
  h_k = h_{k-1} + h tanh(A_k h_{k-1} + B_k u + C_k),  A_k = -R_kᵀR_k - εI, u = h_0.
Flat parameter layout (same as the C-ABI):
  [W_1 (w×(d+1)) b_1 (w) | W_2 (w×w) b_2 | ... | W_L b_L | v (w) | c]
  NAIS-Net blocks: [R_k (w×w) C_k (w) B_k (w×(d+1))] in place of [W_k b_k]

The gradient ∂L/∂Θ goes through ∇ₓu (the loss contains Z_n(Θ)), so it is the
hand-written reverse-over-reverse derivative of the network (shared_grad
below), pinned by central finite differences in tests/test_oracle_shared.py.
"""
import numpy as np

from . import philox
from .bsde import (ALLEN_CAHN, BLACK_SCHOLES, BS_SIGMA, HJB, SIGMA, driver_df_dy, driver_df_dz,
                   driver_f, forward_step, terminal_g)

FC, RESNET, NAIS = 0, 1, 2
NAIS_EPS, NAIS_H = 0.01, 1.0    # A = -RᵀR - εI, block step h (R26)


def num_params(d, w, L, arch=FC):
    blk = w * w + w + (w * (d + 1) if arch == NAIS else 0)
    return w * (d + 1) + w + (L - 1) * blk + w + 1


def unpack(params, d, w, L, arch=FC):
    """Views ([(W_k, b_k) or (R_k, C_k, B_k) for k = 1..L], v, c) into the flat
    vector; layer 1 is always (W_1, b_1), NAIS-Net blocks are (R, C, B)."""
    params = np.asarray(params)
    assert params.shape == (num_params(d, w, L, arch),), (params.shape, num_params(d, w, L, arch))
    layers, off = [], 0
    for k in range(L):
        kin = d + 1 if k == 0 else w
        W = params[off:off + w * kin].reshape(w, kin)
        off += w * kin
        b = params[off:off + w]
        off += w
        if arch == NAIS and k > 0:
            Bk = params[off:off + w * (d + 1)].reshape(w, d + 1)
            off += w * (d + 1)
            layers.append((W, b, Bk))
        else:
            layers.append((W, b))
    v = params[off:off + w]
    c = params[off + w:off + w + 1]
    return layers, v, c


def nais_A(R):
    return -R.T @ R - NAIS_EPS * np.eye(R.shape[0])


def project(params, d, w, L, arch=NAIS):
    """R_k ← R_k((1-ε)/‖R_kᵀR_k‖_F)^½ where ‖RᵀR‖_F > 1-ε (SPEC nets.project_R)."""
    if arch != NAIS:
        return params
    layers, _, _ = unpack(params, d, w, L, arch)
    for lay in layers[1:]:
        R = lay[0]
        f = np.linalg.norm(R.T @ R)
        if f > 1.0 - NAIS_EPS:
            R *= np.sqrt((1.0 - NAIS_EPS) / f)
    return params


def init_params(seed, d, w, L, arch=FC):
    """R23 initialisation, as R7: Xavier-uniform W_k (R_k for NAIS-Net) and v
    (tensor_id 1 + k, and 1 + L for v) from the Philox init stream, NAIS-Net B_k
    Xavier-uniform with tensor 0x100000 + k, zero biases, c ~ U(0, 1) (tensor 0);
    NAIS-Net R_k then projected (R26)."""
    p = np.zeros(num_params(d, w, L, arch))
    layers, v, c = unpack(p, d, w, L, arch)
    for k, lay in enumerate(layers):
        W = lay[0]
        fan_out, fan_in = W.shape
        a = np.sqrt(6.0 / (fan_in + fan_out))
        W[...] = (a * (2.0 * philox.init_uniforms(seed, 1 + k, W.size) - 1.0)).reshape(W.shape)
        if len(lay) == 3:
            Bk = lay[2]
            a = np.sqrt(6.0 / (Bk.shape[0] + Bk.shape[1]))
            Bk[...] = (a * (2.0 * philox.init_uniforms(seed, 0x100000 + k, Bk.size) - 1.0)
                       ).reshape(Bk.shape)
    a = np.sqrt(6.0 / (w + 1))
    v[...] = a * (2.0 * philox.init_uniforms(seed, 1 + L, w) - 1.0)
    c[0] = philox.init_uniforms(seed, 0, 1)[0]
    return project(p, d, w, L, arch)


def forward(params, d, w, L, arch, t, X):
    """u(t, x) for rows (t, X) [R], [R×d]; returns (u [R], cache of h_0..h_L, s_1..s_L).
    NAIS-Net blocks (k ≥ 2): h_k = h_{k-1} + h tanh(A_k h_{k-1} + B_k u + C_k), u = h_0."""
    layers, v, c = unpack(params, d, w, L, arch)
    h = [np.concatenate([np.asarray(t, float).reshape(-1, 1), X], axis=1)]
    s = []
    for k, lay in enumerate(layers):
        if arch == NAIS and k > 0:
            R, C, Bk = lay
            sk = np.tanh(h[-1] @ nais_A(R) + h[0] @ Bk.T + C)
            s.append(sk)
            h.append(h[-1] + NAIS_H * sk)
            continue
        W, b = lay
        sk = np.tanh(h[-1] @ W.T + b)
        s.append(sk)
        h.append(h[-1] + sk if (arch == RESNET and k > 0) else sk)
    return h[-1] @ v + c[0], (h, s)


def input_gradient(params, d, w, L, arch, cache):
    """∇_{(t,x)} u by the chain rule backwards through the layers (the reverse
    pass of autodiff): g_L = v; δ_k = g_k ⊙ (1 - s_k²); g_{k-1} = ρ_k g_k + W_kᵀ δ_k
    with ρ_k = 1 for residual layers.  Returns (g_0 [R×(d+1)], g_1..g_L, δ_1..δ_L)."""
    layers, v, _ = unpack(params, d, w, L, arch)
    h, s = cache
    R = h[0].shape[0]
    g = [None] * (L + 1)
    delta = [None] * (L + 1)
    g[L] = np.broadcast_to(v, (R, w)).copy()
    gu = np.zeros_like(h[0])             # NAIS-Net: the input-injection terms B_kᵀ δ_k
    for k in range(L, 0, -1):
        if arch == NAIS and k > 1:
            Rm, _, Bk = layers[k - 1]
            delta[k] = NAIS_H * g[k] * (1.0 - s[k - 1] ** 2)
            g[k - 1] = g[k] + delta[k] @ nais_A(Rm)
            gu = gu + delta[k] @ Bk
            continue
        W = layers[k - 1][0]
        delta[k] = g[k] * (1.0 - s[k - 1] ** 2)
        g[k - 1] = delta[k] @ W + (g[k] if (arch == RESNET and k > 1) else 0.0)
    g[0] = g[0] + gu
    return g, delta


def grad_g(problem, X):
    """∇g(x) of the terminal conditions (R12, R13): heat and
    Black-Scholes 2x, HJB 2x/(1+|x|²), Allen-Cahn -0.8x/(2+0.4|x|²)²."""
    s = np.sum(X * X, axis=-1, keepdims=True)
    if problem == HJB:
        return 2.0 * X / (1.0 + s)
    if problem == ALLEN_CAHN:
        return -0.8 * X / (2.0 + 0.4 * s) ** 2
    return 2.0 * X


def sigma_t(problem, X, G):
    """z = σ(x)ᵀ ∇ₓu: √2 ∇ₓu, or σ x ⊙ ∇ₓu for Black-Scholes."""
    return BS_SIGMA * X * G if problem == BLACK_SCHOLES else SIGMA * G


def paths(problem, d, N, T, seed, it, m, x0):
    """X_0..X_N [N+1][M×d] and ΔW_0..ΔW_{N-1} (R8 counters, global path ids m)."""
    dt = T / N
    X = [np.full((len(m), d), float(x0))]
    dW = []
    for n in range(N):
        dW.append(philox.brownian_increments(seed, it, n, m, d, dt))
        X.append(forward_step(problem, X[-1], dW[-1]))
    return X, dW


def iteration(problem, d, w, L, arch, N, T, params, seed, it, m, batch_global, x0=0.0, lam=1.0,
              want_grad=True, zN=False):
    """Loss (R24) and its gradient for the shard of global paths m.  Rows are
    (n, m) with n = 0..N; returns dict(loss, loss_sum, grad, r [M×(N+1)], Y, Z).
    zN adds the optional terminal gradient term Σ_m |∇ₓu(t_N, X_N) - ∇g(X_N)|² of
    P:79 (with the paper's Z_N = ∇u, R27)."""
    m = np.asarray(m, dtype=np.int64)
    M = len(m)
    dt = T / N
    X, dW = paths(problem, d, N, T, seed, it, m, x0)
    t = np.repeat(np.arange(N + 1) * dt, M)
    Xr = np.concatenate(X, axis=0)                          # row n·M + j
    u, cache = forward(params, d, w, L, arch, t, Xr)
    g, delta = input_gradient(params, d, w, L, arch, cache)
    Y = u.reshape(N + 1, M)
    Gx = g[0][:, 1:].reshape(N + 1, M, d)                    # ∇ₓu per row
    Z = np.stack([sigma_t(problem, X[n], Gx[n]) for n in range(N + 1)])
    r = np.zeros((N + 1, M))
    for n in range(N):
        r[n] = (Y[n + 1] - Y[n] + driver_f(problem, Y[n], Z[n], lam) * dt
                - np.sum(Z[n] * dW[n], axis=-1))
    r[N] = Y[N] - terminal_g(problem, X[N])
    loss_sum = float(np.sum(r * r))
    eN = Gx[N] - grad_g(problem, X[N]) if zN else None
    if zN:
        loss_sum += float(np.sum(eN * eN))
    out = dict(loss_sum=loss_sum, loss=loss_sum / float(batch_global), r=r, Y=Y, Z=Z)
    if not want_grad:
        return out
    # ---- ∂L/∂Y_n and ∂L/∂z_n (L = Σ r² / B)
    sc = 2.0 / float(batch_global)
    Ybar = np.zeros((N + 1, M))
    Zbar = np.zeros((N + 1, M, d))
    for n in range(N):
        Ybar[n + 1] += sc * r[n]
        Ybar[n] += sc * r[n] * (-1.0 + dt * driver_df_dy(problem, Y[n], Z[n], lam))
        Zbar[n] = sc * r[n][:, None] * (dt * driver_df_dz(problem, Y[n], Z[n], lam) - dW[n])
    Ybar[N] += sc * r[N]
    # ∂L/∂(∇ₓu) = σ(X) z̄ (σ diagonal); no gradient to t
    Gbar = np.concatenate([sigma_t(problem, X[n], Zbar[n]) for n in range(N + 1)], axis=0)
    if zN:   # ∂/∂(∇ₓu) of the Z_N term, rows n = N
        Gbar[N * M:] += sc * eN
    g0bar = np.concatenate([np.zeros((Gbar.shape[0], 1)), Gbar], axis=1)
    out["grad"] = shared_grad(params, d, w, L, arch, cache, g, delta, Ybar.reshape(-1), g0bar)
    return out


def shared_grad(params, d, w, L, arch, cache, g, delta, ubar, g0bar):
    """∂/∂Θ of Σ_rows (ū·u + ḡ_0·g_0): reverse-over-reverse through the input
    gradient, then through the forward pass (R23).

    Adjoint of the input-gradient pass, k = 1..L:
      g_{k-1} = ρ_k g_k + W_kᵀ δ_k :  W̄_k += δ_kᵀ ḡ_{k-1};  δ̄_k = ḡ_{k-1} W_kᵀ;  ḡ_k += ρ_k ḡ_{k-1}
      δ_k = g_k ⊙ (1 - s_k²)       :  ḡ_k += δ̄_k ⊙ (1 - s_k²);  s̄_k = -2 s_k ⊙ g_k ⊙ δ̄_k
      g_L = v                       :  v̄ += Σ ḡ_L
    Adjoint of the forward pass, k = L..1:
      u = v·h_L + c                 :  v̄ += ū h_L;  c̄ += Σ ū;  h̄_L = ū v
      h_k = ρ_k h_{k-1} + s_k       :  s̄_k += h̄_k;  ā_k = s̄_k ⊙ (1 - s_k²)
      a_k = W_k h_{k-1} + b_k       :  W̄_k += ā_kᵀ h_{k-1};  b̄_k += Σ ā_k;  h̄_{k-1} = ρ_k h̄_k + ā_k W_k
    """
    if arch == NAIS:
        return _nais_grad(params, d, w, L, cache, g, delta, ubar, g0bar)
    layers, v, _ = unpack(params, d, w, L)
    h, s = cache
    grad = np.zeros_like(np.asarray(params, dtype=np.float64))
    glayers, gv, gc = unpack(grad, d, w, L)
    res = [arch == RESNET and k > 1 for k in range(L + 1)]   # ρ_k
    gbar = g0bar
    sbar = [None] * (L + 1)
    for k in range(1, L + 1):
        W, _ = layers[k - 1]
        glayers[k - 1][0][...] += delta[k].T @ gbar
        dbar = gbar @ W.T
        sp = 1.0 - s[k - 1] ** 2
        gk_bar = dbar * sp + (gbar if res[k] else 0.0)
        sbar[k] = -2.0 * s[k - 1] * g[k] * dbar
        gbar = gk_bar
    gv[...] += gbar.sum(axis=0)
    gv[...] += ubar @ h[L]
    gc[0] += ubar.sum()
    hbar = np.outer(ubar, v)
    for k in range(L, 0, -1):
        W, _ = layers[k - 1]
        abar = (sbar[k] + hbar) * (1.0 - s[k - 1] ** 2)
        glayers[k - 1][0][...] += abar.T @ h[k - 1]
        glayers[k - 1][1][...] += abar.sum(axis=0)
        if k > 1:
            hbar = abar @ W + (hbar if res[k] else 0.0)
    return grad


def _nais_grad(params, d, w, L, cache, g, delta, ubar, g0bar):
    """Reverse-over-reverse for the NAIS-Net network (R26): layer 1 as FC; block k
    (A_k = -R_kᵀR_k - εI symmetric, u = h_0):
      input-gradient adjoint, k = 1..L, seed ḡ_u = g0bar:
        layer 1: W̄_1 += δ_1ᵀ ḡ_u;  δ̄_1 = ḡ_u W_1ᵀ;  ḡ_1 = δ̄_1 ⊙ s'_1;  s̄_1 = -2 s_1 g_1 δ̄_1
        block k: Ā_k += δ_kᵀ ḡ_{k-1};  B̄_k += δ_kᵀ ḡ_u;  δ̄_k = ḡ_{k-1} A_k + ḡ_u B_kᵀ;
                 ḡ_k = ḡ_{k-1} + h δ̄_k ⊙ s'_k;  s̄_k = -2 h s_k g_k δ̄_k
      forward adjoint, k = L..1: ā_k = (s̄_k + h h̄_k) ⊙ s'_k (h = 1 for layer 1);
        block: Ā_k += ā_kᵀ h_{k-1}, B̄_k += ā_kᵀ u, C̄_k += Σ ā_k, h̄_{k-1} = h̄_k + ā_k A_k;
        layer 1: W̄_1 += ā_1ᵀ u, b̄_1 += Σ ā_1
      then R̄_k = -R_k(Ā_k + Ā_kᵀ)."""
    layers, v, _ = unpack(params, d, w, L, NAIS)
    h, s = cache
    grad = np.zeros_like(np.asarray(params, dtype=np.float64))
    glayers, gv, gc = unpack(grad, d, w, L, NAIS)
    Abar = [None] + [np.zeros((w, w)) for _ in range(1, L)]
    gu_bar = g0bar
    sbar = [None] * (L + 1)
    W1 = layers[0][0]
    glayers[0][0][...] += delta[1].T @ gu_bar
    db = gu_bar @ W1.T
    sp = 1.0 - s[0] ** 2
    gbar = db * sp
    sbar[1] = -2.0 * s[0] * g[1] * db
    for k in range(2, L + 1):
        Rm, C, Bk = layers[k - 1]
        A = nais_A(Rm)
        Abar[k - 1] += delta[k].T @ gbar
        glayers[k - 1][2][...] += delta[k].T @ gu_bar
        db = gbar @ A + gu_bar @ Bk.T
        sp = 1.0 - s[k - 1] ** 2
        sbar[k] = -2.0 * NAIS_H * s[k - 1] * g[k] * db
        gbar = gbar + NAIS_H * db * sp
    gv[...] += gbar.sum(axis=0)
    gv[...] += ubar @ h[L]
    gc[0] += ubar.sum()
    hbar = np.outer(ubar, v)
    for k in range(L, 0, -1):
        sp = 1.0 - s[k - 1] ** 2
        if k > 1:
            Rm, C, Bk = layers[k - 1]
            abar = (sbar[k] + NAIS_H * hbar) * sp
            Abar[k - 1] += abar.T @ h[k - 1]
            glayers[k - 1][2][...] += abar.T @ h[0]
            glayers[k - 1][1][...] += abar.sum(axis=0)
            hbar = hbar + abar @ nais_A(Rm)
        else:
            abar = (sbar[1] + hbar) * sp
            glayers[0][0][...] += abar.T @ h[0]
            glayers[0][1][...] += abar.sum(axis=0)
    for k in range(1, L):
        Rm = layers[k][0]
        glayers[k][0][...] = -Rm @ (Abar[k] + Abar[k].T)
    return grad


def u0(params, d, w, L, arch, x0):
    """Y0 = u(0, X_0) with X_0 = x0·1 (the quantity bsde_y0 returns)."""
    u, _ = forward(params, d, w, L, arch, np.zeros(1), np.full((1, d), float(x0)))
    return float(u[0])
