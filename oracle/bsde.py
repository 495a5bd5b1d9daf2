"""Per-step-network deep-BSDE iteration in float64 (TEST INFRASTRUCTURE ONLY).

What one training iteration computes (the hot path that BASELINE.json's
north_star names; formulation = the Han et al. scheme the paper describes at
P:78, "there are N different neural networks. Y0 and Z0 are treated as
parameters and all the Y_n are computed using an Euler discretization"):

  ΔW_n ~ N(0, Δt)                                  Eq. 5, P:64   (philox.py, R8)
  X_{n+1} = X_n + σ ΔW_n,  σ = √2 I, μ = 0         Eq. 5; Eq. 12
     (Black-Scholes: X_{n+1} = X_n + σ X_n ⊙ ΔW_n, σ(x) = 0.4 diag(x); R21)
  Z_n = net_n(X_n)  (lift, one residual block, head) Eq. 7; R4
  Y_{n+1} = Y_n + φ Δt + Z_n·ΔW_n,  φ = -f         Eq. 5; R2
  L = (1/B) Σ_m (Y_N - g(X_N))²                    Eq. 6, P:75 (terminal term); R5
  gradient by the hand-derived adjoint (no autograd)   R19/DESIGN.md §Adjoint
  Adam                                             P:319; R6
  multilevel prolongation N -> 2N                  §3.2; R14

Flat parameter layout (R-layout, same as the C-ABI, include/bsde.h):
  [Y0 | step 0: W1 (w×d) b1 (w) W2 (w×w) b2 (w) W3 (d×w) b3 (d) | step 1 ...]
all row-major.
"""
import numpy as np

from . import philox

HEAT, HJB, ALLEN_CAHN, BLACK_SCHOLES = 0, 1, 2, 3
PROBLEM_NAMES = {"heat": HEAT, "hjb": HJB, "allen_cahn": ALLEN_CAHN,
                 "black_scholes": BLACK_SCHOLES}
SIGMA = np.sqrt(2.0)          # dX = √2 dW in every config (BASELINE.json configs 1-5)
# Black-Scholes: uncorrelated assets with the
# same volatility, "d = 100, r = 0.05 and σ = 0.4", g(x) = ‖x‖².
BS_RATE, BS_SIGMA = 0.05, 0.4


def forward_step(problem, X, dW):
    """Euler step of the forward SDE (Eq. 5; μ = 0): X + σ ΔW with σ = √2 I,
    or for Black-Scholes X + σ X ⊙ ΔW (σ(x) = σ diag(x))."""
    if problem == BLACK_SCHOLES:
        return X + BS_SIGMA * X * dW
    return X + SIGMA * dW


# ----------------------------------------------------------------------------
# Problem data (R2, R10-R13).  Driver in the Han convention:
#   Y_{n+1} = Y_n - f(Y_n, Z_n) Δt + Z_n·ΔW_n
# ----------------------------------------------------------------------------
def driver_f(problem, y, z, lam=1.0):
    """f(y, z): heat 0 (R13); HJB -λ|z|²/2 (P:302 read as ‖Du‖², R10);
    Allen-Cahn y - y³ (R12); Black-Scholes -r(y - Σ_i z_i / σ) (P:293 with
    z = σᵀ∇u = σ x ⊙ ∇u, so (Du)ᵀx = Σ z_i / σ; R21)."""
    if problem == HEAT:
        return np.zeros_like(y)
    if problem == HJB:
        return -0.5 * lam * np.sum(z * z, axis=-1)
    if problem == ALLEN_CAHN:
        return y - y ** 3
    if problem == BLACK_SCHOLES:
        return -BS_RATE * (y - np.sum(z, axis=-1) / BS_SIGMA)
    raise ValueError(problem)


def driver_df_dy(problem, y, z, lam=1.0):
    if problem == ALLEN_CAHN:
        return 1.0 - 3.0 * y * y
    if problem == BLACK_SCHOLES:
        return np.full_like(y, -BS_RATE)
    return np.zeros_like(y)


def driver_df_dz(problem, y, z, lam=1.0):
    if problem == HJB:
        return -lam * z
    if problem == BLACK_SCHOLES:
        return np.full_like(z, BS_RATE / BS_SIGMA)
    return np.zeros_like(z)


def terminal_g(problem, x):
    """g: heat |x|² (R13); HJB ln(0.5(1+|x|²)); Allen-Cahn 1/(2+0.4|x|²) (R12);
    Black-Scholes |x|²."""
    s = np.sum(x * x, axis=-1)
    if problem in (HEAT, BLACK_SCHOLES):
        return s
    if problem == HJB:
        return np.log(0.5 * (1.0 + s))
    if problem == ALLEN_CAHN:
        return 1.0 / (2.0 + 0.4 * s)
    raise ValueError(problem)


# ----------------------------------------------------------------------------
# Parameters
# ----------------------------------------------------------------------------
def step_size(d, w):
    """P_step = 2dw + w² + 2w + d."""
    return 2 * d * w + w * w + 2 * w + d


def num_params(d, w, N):
    return 1 + N * step_size(d, w)


def unpack(params, d, w, N):
    """Views (Y0, [dict(W1,b1,W2,b2,W3,b3) for n < N]) into the flat vector."""
    params = np.asarray(params)
    assert params.shape == (num_params(d, w, N),), (params.shape, num_params(d, w, N))
    nets = []
    off = 1
    for _ in range(N):
        net = {}
        for name, shape in (("W1", (w, d)), ("b1", (w,)), ("W2", (w, w)),
                            ("b2", (w,)), ("W3", (d, w)), ("b3", (d,))):
            size = int(np.prod(shape))
            net[name] = params[off:off + size].reshape(shape)
            off += size
        nets.append(net)
    return params[0:1], nets


def init_params(seed, d, w, N, zero_head=False):
    """R7: Xavier-uniform W ~ U(-a, a), a = sqrt(6/(fan_in+fan_out)); biases 0;
    Y0 ~ U(0, 1).  Uniforms from the Philox init stream, tensor_id = 1 + 3n + k
    (k = 0, 1, 2 for W1, W2, W3) and 0 for Y0.  zero_head (R7b, Allen-Cahn):
    W3 = 0, so Z ≡ 0 at initialisation."""
    p = np.zeros(num_params(d, w, N))
    y0, nets = unpack(p, d, w, N)
    y0[0] = philox.init_uniforms(seed, 0, 1)[0]
    for n, net in enumerate(nets):
        for k, name in enumerate(("W1", "W2") if zero_head else ("W1", "W2", "W3")):
            fan_out, fan_in = net[name].shape
            a = np.sqrt(6.0 / (fan_in + fan_out))
            u = philox.init_uniforms(seed, 1 + 3 * n + k, net[name].size)
            net[name][...] = (a * (2.0 * u - 1.0)).reshape(net[name].shape)
    return p


def round_bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float64 (R17 diagnosis mode)."""
    f = np.asarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def round_fp16(x):
    """Round-to-nearest-even to IEEE binary16 (via fp32), returned as float64:
    the storage precision of ΔW_n in the tensor-core reading of R17."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float64)


def _ident(a):
    return a


# ----------------------------------------------------------------------------
# One iteration: rollout + terminal loss + hand adjoint
# ----------------------------------------------------------------------------
def net_forward(net, x, bf16=False, tc=False, rb=round_bf16):
    """Per-step Z-net (R4; Eq. 7 with h = 1):
    A1 = W1 x + b1, H1 = ReLU(A1), A2 = W2 H1 + b2, H2 = H1 + ReLU(A2), Z = W3 H2 + b3.

    bf16 (R17 as SURVEY states it): GEMM operands rounded to bf16, everything
    else exact.  tc (R17 as DESIGN.md records it for the tensor-core path): the
    biases are GEMM operands too (folded into a constant-1 input column), H1 is
    stored as bf16(ReLU(A1)) and the residual sum is formed in bf16,
    H2 = bf16(H1 + bf16(ReLU(A2))) (one rounding of the exact sum of two bf16
    values).  ``rb`` is the rounding (identity in the structural pin)."""
    if tc:
        A1 = rb(x) @ rb(net["W1"]).T + rb(net["b1"])
        H1 = rb(np.maximum(A1, 0.0))
        A2 = H1 @ rb(net["W2"]).T + rb(net["b2"])
        H2 = rb(H1 + rb(np.maximum(A2, 0.0)))
        Z = H2 @ rb(net["W3"]).T + rb(net["b3"])
        return A1, H1, A2, H2, Z
    op = round_bf16 if bf16 else _ident
    A1 = op(x) @ op(net["W1"]).T + net["b1"]
    H1 = np.maximum(A1, 0.0)
    A2 = op(H1) @ op(net["W2"]).T + net["b2"]
    H2 = H1 + np.maximum(A2, 0.0)
    Z = op(H2) @ op(net["W3"]).T + net["b3"]
    return A1, H1, A2, H2, Z


def iteration(problem, d, w, N, T, params, seed, it, paths, batch_global,
              x0=0.0, lam=1.0, want_grad=True, bf16=False, keep=False, kink_band=0.0,
              mask_shift=0.0, coupled_factor=1, tc=False, rb=round_bf16, rh=round_fp16,
              kink_flip=0.0):
    """One training iteration on the shard ``paths`` (global path indices).

    Returns dict(loss_sum=Σ_m R², loss=Σ R²/B_global, grad=∂L/∂params of this
    shard's contribution (sums over shards to the full gradient, R5, §8(e)),
    R, Y_N, X_N, and per-step traces if keep).

    kink_band > 0 also returns ``slack`` (shape of grad): for every hidden unit
    whose pre-activation lies within kink_band·(Σ|W x| + |b|) of the ReLU kink,
    both masks are valid answers of a finite-precision evaluation (R15, R19),
    and slack bounds (to first order) how much the gradient moves when that
    mask flips.  mask_shift (tests only) evaluates the backward masks as
    1[A > mask_shift] to emulate such flips.  coupled_factor = f > 1 draws every
    increment as the sum of the f increments of the grid with N·f steps that it
    spans (coupled multilevel paths, philox.coupled_increments).  kink_flip > 0
    widens that band by kink_flip·max_j |W_ij x_j| (the largest single term of the
    pre-activation): the reach of one operand x_j landing on the other side of a
    rounding boundary (one bf16 ulp, kink_flip = 2^-8), which finite-precision
    accumulation can cause upstream of the kink (R19, tensor-core reading).
    """
    paths = np.asarray(paths, dtype=np.int64)
    B = float(batch_global)
    dt = T / N
    y0, nets = unpack(params, d, w, N)
    M = paths.shape[0]
    X = np.full((M, d), float(x0))
    Y = np.full(M, y0[0])
    trace = []
    for n in range(N):
        dW = (philox.brownian_increments(seed, it, n, paths, d, dt) if coupled_factor == 1
              else philox.coupled_increments(seed, it, n, paths, d, dt, coupled_factor))
        A1, H1, A2, H2, Z = net_forward(nets[n], X, bf16, tc, rb)        # P:78, Eq. 7
        trace.append((X, dW, A1, H1, A2, H2, Z, Y))
        dWz = rh(dW) if tc else dW
        Y = Y - driver_f(problem, Y, Z, lam) * dt + np.sum(Z * dWz, axis=-1)  # P:66 (φ=-f)
        X = forward_step(problem, X, dW)
    R = Y - terminal_g(problem, X)
    out = dict(loss_sum=float(np.sum(R * R)), loss=float(np.sum(R * R) / B),
               R=R, Y_N=Y, X_N=X)
    if keep:
        out["trace"] = trace
    if not want_grad:
        return out
    # Adjoint: ā_N = ∂L/∂Y_N = 2R/B.
    grad = np.zeros_like(np.asarray(params, dtype=np.float64))
    gy0, gnets = unpack(grad, d, w, N)
    if kink_band > 0.0:
        slack = np.zeros_like(grad)
        _, snets = unpack(slack, d, w, N)
    abar = 2.0 * R / B
    op = round_bf16 if bf16 else (lambda a: a)
    for n in range(N - 1, -1, -1):
        X, dW, A1, H1, A2, H2, Z, Yn = trace[n]
        net, g = nets[n], gnets[n]
        # ∂Y_{n+1}/∂Z_n = ΔW_n - Δt ∂_z f ;  ∂Y_{n+1}/∂Y_n = 1 - Δt ∂_y f
        dZ = abar[:, None] * ((rh(dW) if tc else dW) - dt * driver_df_dz(problem, Yn, Z, lam))
        m2 = A2 > mask_shift                         # ReLU'(0) = 0 (R15)
        m1 = A1 > mask_shift
        if tc:
            dZ = rb(dZ)
            g["W3"][...] = dZ.T @ H2
            g["b3"][...] = dZ.sum(0)
            dH2 = dZ @ rb(net["W3"])
            dA2 = rb(dH2) * m2
            g["W2"][...] = dA2.T @ H1
            g["b2"][...] = dA2.sum(0)
            dH1 = dH2 + dA2 @ rb(net["W2"])
            dA1 = rb(dH1) * m1
            g["W1"][...] = dA1.T @ rb(X)
            g["b1"][...] = dA1.sum(0)
        else:
            g["W3"][...] = op(dZ).T @ op(H2)
            g["b3"][...] = dZ.sum(0)
            dH2 = op(dZ) @ op(net["W3"])
            dA2 = dH2 * m2
            g["W2"][...] = op(dA2).T @ op(H1)
            g["b2"][...] = dA2.sum(0)
            dH1 = dH2 + op(dA2) @ op(net["W2"])
            dA1 = dH1 * m1
            g["W1"][...] = op(dA1).T @ op(X)
            g["b1"][...] = dA1.sum(0)
        if kink_band > 0.0:
            s = snets[n]
            amb1 = np.abs(A1) <= (kink_band * (np.abs(X) @ np.abs(net["W1"]).T + np.abs(net["b1"]))
                                  + kink_flip * _max_term(X, net["W1"]))
            amb2 = np.abs(A2) <= (kink_band * (np.abs(H1) @ np.abs(net["W2"]).T + np.abs(net["b2"]))
                                  + kink_flip * _max_term(H1, net["W2"]))
            e2 = np.abs(dH2) * amb2                  # |ΔdA2| if an A2 mask flips
            e1 = (np.abs(dH1) * amb1                 # |ΔdA1| from an A1 flip ...
                  + (e2 @ np.abs(net["W2"])) * (m1 | amb1))   # ... or propagated from A2
            s["W2"][...] = e2.T @ np.abs(H1)
            s["b2"][...] = e2.sum(0)
            s["W1"][...] = e1.T @ np.abs(X)
            s["b1"][...] = e1.sum(0)
        abar = abar * (1.0 - dt * driver_df_dy(problem, Yn, Z, lam))
    gy0[0] = abar.sum()
    out["grad"] = grad
    if kink_band > 0.0:
        out["slack"] = slack
    return out


def _max_term(x, W):
    """max_j |W_ij x_j| per (row of x, i), or 0 when the caller passes no flip width."""
    out = np.empty((x.shape[0], W.shape[0]))
    aW = np.abs(W)
    for i in range(0, x.shape[0], 128):
        out[i:i + 128] = np.max(np.abs(x[i:i + 128])[:, None, :] * aW[None], axis=2)
    return out


def loss_and_grad(problem, d, w, N, T, params, seed, it, batch, **kw):
    """Full-batch iteration over global paths 0..batch-1."""
    return iteration(problem, d, w, N, T, params, seed, it, np.arange(batch), batch, **kw)


# ----------------------------------------------------------------------------
# Adam ("Adam optimizer"; hyper-parameters R6) with the divergence guard
# (SPEC S:425 reading: loss > 1e12 or non-finite -> skip the update).
# ----------------------------------------------------------------------------
class AdamState:
    def __init__(self, n):
        self.m = np.zeros(n)
        self.v = np.zeros(n)
        self.t = 0


def adam_step(params, grad, state, lr, beta1=0.9, beta2=0.999, eps=1e-8, loss=0.0):
    """θ ← θ - lr m̂/(√v̂ + ε), m̂ = m/(1-β1^t), v̂ = v/(1-β2^t), t counted from 1.
    Returns False (and leaves everything untouched) on divergence."""
    if not (np.isfinite(loss) and loss <= 1e12 and np.all(np.isfinite(grad))):
        return False
    state.t += 1
    state.m = beta1 * state.m + (1.0 - beta1) * grad
    state.v = beta2 * state.v + (1.0 - beta2) * grad * grad
    mhat = state.m / (1.0 - beta1 ** state.t)
    vhat = state.v / (1.0 - beta2 ** state.t)
    params -= lr * mhat / (np.sqrt(vhat) + eps)
    return True


# ----------------------------------------------------------------------------
# Multilevel prolongation (§3.2: h_l = h0 M^-l with M = 2; R14)
# ----------------------------------------------------------------------------
COPY, INTERP = 0, 1


def prolongate(params, d, w, N, mode=COPY):
    """θ^{2N}_k = θ^N_{k//2} (copy), or θ_{2n} = θ_n, θ_{2n+1} = (θ_n+θ_{n+1})/2
    for n < N-1 and θ_{2N-1} = θ_{N-1} (interp).  Y0 is carried (R14)."""
    P = step_size(d, w)
    src = np.asarray(params)[1:].reshape(N, P)
    dst = np.empty((2 * N, P))
    if mode == COPY:
        dst[0::2] = src
        dst[1::2] = src
    else:
        dst[0::2] = src
        dst[1:-1:2] = 0.5 * (src[:-1] + src[1:])
        dst[-1] = src[-1]
    return np.concatenate([np.asarray(params)[:1], dst.reshape(-1)])


# ----------------------------------------------------------------------------
# Training loops (host schedule; §3.2 multilevel; R9 fresh paths every iteration)
# ----------------------------------------------------------------------------
def train(problem, d, w, N, T, params, seed, batch, iters, lr, it0=0, state=None, lam=1.0):
    state = state or AdamState(params.size)
    losses = []
    for k in range(iters):
        r = loss_and_grad(problem, d, w, N, T, params, seed, it0 + k, batch, lam=lam)
        adam_step(params, r["grad"], state, lr, loss=r["loss"])
        losses.append(r["loss"])
    return params, state, losses


def prolongate_adam(state, d, w, N, mode=COPY):
    """R14b: the moments m, v follow the parameters' prolongation rule
    (the same function, `prolongate`), t is kept; the alternative to the R14 reset."""
    out = AdamState(1 + 2 * N * step_size(d, w))
    out.m = prolongate(state.m, d, w, N, mode)
    out.v = prolongate(state.v, d, w, N, mode)
    out.t = state.t
    return out


def train_multilevel(problem, d, w, levels, T, params, seed, batch, iters_per_level, lr,
                     mode=COPY, lam=1.0, keep_adam=False):
    """Levels N_0 < N_1 = 2N_0 < ...; Adam state reset at each change (R14), or
    prolonged with the parameters (keep_adam, R14b); the Philox iteration counter
    continues across levels (R9)."""
    it = 0
    history = []
    state = None
    for li, N in enumerate(levels):
        if li:
            params = prolongate(params, d, w, levels[li - 1], mode)
            state = prolongate_adam(state, d, w, levels[li - 1], mode) if keep_adam else None
        params, state, losses = train(problem, d, w, N, T, params, seed, batch,
                                      iters_per_level[li], lr, it0=it, state=state, lam=lam)
        history += [(li, N, l) for l in losses]
        it += iters_per_level[li]
    return params, history
