// shared.cu — the paper's own formulation (PAPER.md:69-77,
// fig:neural, Eq. 6): ONE network u(t, x; Θ) for every time step, Y_n =
// u(t_n, X_n), z_n = σ(X_n)ᵀ∇ₓu(t_n, X_n), and the residual-sum loss
//   L = (1/B) Σ_m [ Σ_{n<N} (Y_{n+1} - Y_n + f(Y_n, z_n)Δt - z_n·ΔW_n)² + (Y_N - g(X_N))² ]
// (R23, R24).  Because the loss contains ∇ₓu, ∂L/∂Θ is a second derivative of
// the network: the hand-written reverse-over-reverse pass below, checked
// against oracle/shared.py (itself pinned by finite differences).
//
// Every (path, time) pair is an independent row once the paths are drawn (X
// does not depend on Θ), so the iteration is a sequence of row-batched dense
// GEMMs over R = (N+1)·B_local rows with fused elementwise epilogues:
//
//   paths     U0 = [t_n | X_n] rows, ΔW_n                    (Philox, Euler; R8)
//   forward   a_k = h_{k-1} W_kᵀ + b_k, s_k = tanh a_k, h_k = s_k (+ h_{k-1}, ResNet)   NT GEMMs
//             δ_L = v ⊙ (1 - s_L²)                              (last epilogue)
//   ∇ₓu       g_{k-1} = δ_k W_k (+ g_k), δ_{k-1} = g_{k-1} ⊙ (1 - s_{k-1}²)            NN GEMMs
//   rows      u = v·h_L + c; z = σ(X)ᵀ g_0[1:]; z·ΔW, |z|², Σz                  (warp per row)
//   loss      r_n, Σ r²; ū = ∂L/∂u, ḡ_0 = σ(X) z̄ per row                          (warp per row)
//   up        W̄_k += δ_kᵀ ḡ_{k-1};  δ̄_k = ḡ_{k-1} W_kᵀ;  ḡ_k = δ̄_k ⊙ s'_k (+ ḡ_{k-1});
//             s̄_k = -2 s_k g_k δ̄_k                                      NT + TN GEMMs
//   down      ā_k = (s̄_k + h̄_k) ⊙ s'_k;  W̄_k += ā_kᵀ h_{k-1}, b̄_k += Σ ā_k;
//             h̄_{k-1} = ā_k W_k (+ h̄_k)                                   NN + TN GEMMs
//   head      v̄ = Σ (ḡ_L + ū h_L), c̄ = Σ ū
//
// Precision FP32 (the paper's PyTorch precision): SIMT FFMA GEMMs,
// 128×128×8 tiles with 8×8 register tiles per thread (double-buffered smem) when
// the grid fills ≥ 2 waves, else 64×64×16 with 4×4; weight gradients split the
// row reduction over CTAs (fp32 atomics) and fold the bias sums in.  Precision
// BF16 (FC / ResNet): the row GEMMs run on tcgen05 (k_tc_rowgemm, bf16 operands,
// fp32 TMEM accumulation, same epilogues); the weight gradients stay fp32.
// NAIS-Net blocks (arch 2): A_k = -R_kᵀR_k - εI per iteration, the input
// injection as a second operand pair of the row GEMMs (R26).
#include <type_traits>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace bsde {
namespace {

#define RET(x)                                \
  do {                                        \
    cudaError_t e_ = (x);                     \
    if (e_ != cudaSuccess) return e_;         \
  } while (0)

constexpr int TB = 64, TK = 16, NTH = 256;

// ---------------------------------------------------------------- GEMM cores
// An optional second operand pair accumulated into the same outputs (same NT/NN
// mode): C = A·B' + A2·B2' (NAIS-Net: h A_kᵀ + u B_kᵀ, ḡ A_k + ḡ_u B_kᵀ).
struct Op2 {
  const float* A = nullptr;
  int lda = 0;
  const float* B = nullptr;
  int ldb = 0, K = 0;
};
// Row GEMM: C[i][j] = Σ_k A[i][k]·B'[k][j] for i < R, j < NC, then epi(i, j, c).
// NT: B' = Bᵀ with B row-major [NC×K] (a weight W_k [out×in]);  NN: B' = B, [K×NC].
template <bool NT, class Epi>
__global__ void __launch_bounds__(NTH) k_gemm_rows(const float* __restrict__ A, int lda,
                                                   const float* __restrict__ B, int ldb, int R,
                                                   int NC, int K, Epi epi, Op2 op2) {
  const float* Ap = A;
  const float* Bp = B;
  int ldap = lda, ldbp = ldb, Kp = K;
  __shared__ __align__(16) float As[2][TK][TB + 4];
  __shared__ __align__(16) float Bs[2][TK][TB + 4];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int i0 = blockIdx.y * TB, j0 = blockIdx.x * TB;
  float ra[4], rb[4];   // the next k-tile, in registers while the current one is used
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = t + NTH * e, ii = idx >> 4, kk = idx & 15;
      const int i = i0 + ii, k = k0 + kk;
      ra[e] = (i < R && k < Kp) ? __ldg(Ap + (int64_t)i * ldap + k) : 0.0f;
      if (NT) {
        const int j = j0 + ii;
        rb[e] = (j < NC && k < Kp) ? __ldg(Bp + (int64_t)j * ldbp + k) : 0.0f;
      } else {
        const int kb = idx >> 6, jj = idx & 63, k2 = k0 + kb, j = j0 + jj;
        rb[e] = (k2 < Kp && j < NC) ? __ldg(Bp + (int64_t)k2 * ldbp + j) : 0.0f;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = t + NTH * e, ii = idx >> 4, kk = idx & 15;
      As[buf][kk][ii] = ra[e];
      if (NT) Bs[buf][kk][ii] = rb[e];
      else Bs[buf][idx >> 6][idx & 63] = rb[e];
    }
  };
  float acc[4][4] = {};
  for (int pass = 0; pass < (op2.A ? 2 : 1); ++pass) {
  if (pass) { Ap = op2.A; Bp = op2.B; ldap = op2.lda; ldbp = op2.ldb; Kp = op2.K; }
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < Kp; k0 += TK) {
    const bool more = k0 + TK < Kp;
    if (more) load(k0 + TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[buf][kk][4 * ty]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][kk][4 * tx]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  }   // pass
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = i0 + 4 * ty + r, j = j0 + 4 * tx;
    if (i >= R) continue;
    if (epi.ld % 4 == 0 && j + 3 < NC) {
      epi.v4(i, j, make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]));
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (j + c < NC) epi(i, j + c, acc[r][c]);
    }
  }
}

// ---------------------------------------------------------------- tcgen05 row GEMM
// bf16 operands, fp32 TMEM accumulation (BSDE_BF16 precision of the shared
// formulation).  One CTA = 128 rows of C[R×NC] = A[R×K]·W_kᵀ (NT) or A·W_k (NN);
// W_k's bf16 image [w rows × Kp cols] (tc_common.cuh layout) sits in shared
// memory whole (NT: K-major B, NN: MN-major B — the same image), A is converted
// from fp32 to bf16 64 columns at a time into a double-buffered image; thread 0
// issues the MMAs; the 4 warps read the accumulator (lane = row) for the epilogue.
constexpr int TCK = 64;   // K chunk of the A image
#ifndef BSDE_EXP_TCN
#define BSDE_EXP_TCN 128
#endif
constexpr int TCN = BSDE_EXP_TCN;  // N tile (columns of C per CTA)
template <bool NT, class Epi, int TN>
__global__ void __launch_bounds__(256, TN <= 128 ? 2 : 1) k_tc_rowgemm(const float* __restrict__ A, int lda, int R,
                                                      int K, const uint16_t* __restrict__ wimg,
                                                      int wrows, int Kp, int NC, int Npad,
                                                      Epi epi) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* abuf = sm;                                   // 2 × [128 × TCK] bf16
  uint8_t* wsm = sm + 2 * 128 * TCK * 2;                // this CTA's slab of the weight image
  __shared__ __align__(8) uint64_t bars[3];             // weights, MMA done (×2)
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // blockIdx.x = N tile (fastest): the CTAs sharing a row tile run back to back, so the
  // second one finds A in L2
  const int i0 = blockIdx.y * 128, n0 = blockIdx.x * TN, nn = min(TN, Npad - n0);
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, TN);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(wimg);
  if (t == 0) {   // NT: image rows [n0, n0+nn) are contiguous; NN: columns [n0, n0+nn) of every row group
    if (NT) {
      const uint32_t bytes = (uint32_t)nn * Kp * 2;
      mbar_expect_tx(&bars[0], bytes);
      const uint8_t* src = wsrc + (size_t)(n0 / 8) * (Kp * 16);
      for (uint32_t off = 0; off < bytes; off += 16384u)
        bulk_g2s(wsm + off, src + off, min(16384u, bytes - off), &bars[0]);
    } else {
      const uint32_t gbytes = (uint32_t)nn * 16;
      mbar_expect_tx(&bars[0], gbytes * (uint32_t)(wrows / 8));
      for (int g = 0; g < wrows / 8; ++g)
        bulk_g2s(wsm + g * gbytes, wsrc + (size_t)g * (Kp * 16) + (n0 / 8) * 128, gbytes, &bars[0]);
    }
  }
  const int Kg = (K + 15) / 16 * 16;                     // GEMM K, padded
  const int nch = (Kg + TCK - 1) / TCK;
  // chunk kc of A (fp32, row-major) -> bf16 image in buffer b: 16 threads per row,
  // 4 consecutive columns each (coalesced 256-byte row segments), 8 rows per pass
  auto convert = [&](int kc, int b) {
    const int k0 = kc * TCK, cw = min(TCK, Kg - k0), c4 = 4 * (t & 15);
    uint8_t* img = abuf + b * (128 * TCK * 2);
    if (c4 >= cw) return;
    // all 8 rows' loads first (independent, in flight together), then convert
    float4 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = i0 + (t >> 4) + 16 * q, k = k0 + c4;
      v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < R) {
        const float* src = A + (int64_t)i * lda + k;
        if (k + 3 < K) {
          v[q] = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          if (k < K) v[q].x = __ldg(src);
          if (k + 1 < K) v[q].y = __ldg(src + 1);
          if (k + 2 < K) v[q].z = __ldg(src + 2);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = (t >> 4) + 16 * q;
      const uint2 u = make_uint2(pack2(v[q].x, v[q].y), pack2(v[q].z, v[q].w));
      *reinterpret_cast<uint2*>(img + (r >> 3) * (cw * 16) + (c4 >> 3) * 128 + (r & 7) * 16 +
                                (c4 & 7) * 2) = u;
    }
  };
  const uint32_t idesc = idesc_bf16(128, nn, false, !NT);
  convert(0, 0);
  fence_async_smem();
  tc_before();
  __syncthreads();
  for (int kc = 0; kc < nch; ++kc) {
    const int b = kc & 1, cw = min(TCK, Kg - kc * TCK);
    if (t == 0) {
      tc_after();
      if (kc == 0) mbar_wait(&bars[0], 0);
      const Opnd a = kmaj(abuf + b * (128 * TCK * 2), cw);
      Opnd w = NT ? kmaj(wsm, Kp) : mnmaj(wsm, nn);
      w.base += NT ? (uint32_t)kc * (TCK / 8) * 128u : (uint32_t)kc * (TCK / 8) * (uint32_t)nn * 16u;
      gemm(tm, a, w, cw / 16, idesc, kc > 0);
      mma_commit(&bars[1 + b]);
    }
    if (kc + 1 < nch) {
      if (kc >= 1) mbar_wait(&bars[1 + (b ^ 1)], (uint32_t)(((kc - 1) >> 1) & 1));   // chunk kc-1 read it
      convert(kc + 1, b ^ 1);
      fence_async_smem();
    }
    tc_before();
    __syncthreads();
  }
  mbar_wait(&bars[1 + ((nch - 1) & 1)], (uint32_t)(((nch - 1) >> 1) & 1));
  tc_after();
  // epilogue, two phases through shared memory (the operand buffers are free now):
  // TMEM -> smem tile [128 rows][nn] (lane = row, warps 0-3 / 4-7 split the column
  // groups), then each warp walks whole rows with 4 columns per lane, so every
  // epilogue array access is a coalesced row segment
  float* stile = reinterpret_cast<float*>(sm);
  const int ldt = nn + 4;
  {
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_base = tm + ((uint32_t)((warp & 3) * 32) << 16);
    const int ngrp = nn / 16, gsplit = (ngrp + 1) / 2;
    const int jb = (warp < 4 ? 0 : gsplit) * 16, je = (warp < 4 ? gsplit : ngrp) * 16;
    for (int jl = jb; jl < je; jl += 16) {
      float v[16];
      tmem_ld16(lane_base + (uint32_t)jl, v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(stile + row * ldt + jl + 4 * q) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  __syncthreads();
  for (int r = warp; r < 128; r += 8) {
    const int i = i0 + r, jl = 4 * lane;
    if (i >= R || jl >= nn) continue;
    const float4 val = *reinterpret_cast<const float4*>(stile + r * ldt + jl);
    const int j = n0 + jl;
    if (epi.ld % 4 == 0 && j + 3 < NC) {
      epi.v4(i, j, val);
    } else {
      const float vv[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j + e < NC) epi(i, j + e, vv[e]);
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, TN);
  }
}

// tcgen05 weight-gradient GEMM: C[P×Q] += Σ_r A[r][p]·B[r][q] over this CTA's row
// range (split-K over blockIdx.z, fp32 atomics), bf16 operands, fp32 TMEM
// accumulation.  One CTA = 128 p (MMA M) × Qt ≤ 256 q (MMA N); both operands are
// MN-major images of 32 path-rows (K) converted from fp32, double-buffered.
// bias (blockIdx.y == 0... CTAs of q-tile 0): += Σ_r A[r][p] accumulated during conversion.
constexpr int TNK = 32;   // rows (K) per chunk
__global__ void __launch_bounds__(256, 2) k_tc_tngemm(const float* __restrict__ A, int lda,
                                                     const float* __restrict__ B, int ldb, int R,
                                                     int P, int Q, float* __restrict__ C, int ldc,
                                                     float* __restrict__ bias, int rows_per_split,
                                                     int Qt) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t sm[];
  const int Qtp = (Qt + 15) / 16 * 16;
  uint8_t* aimg = sm;                                   // 2 × [TNK rows × 128 cols] bf16
  uint8_t* bimg = sm + 2 * TNK * 128 * 2;               // 2 × [TNK rows × Qtp cols] bf16
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tslot;
  __shared__ float bsum[128];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int p0 = blockIdx.x * 128, q0 = blockIdx.y * Qt;
  const int r_begin = blockIdx.z * rows_per_split, r_end = min(R, r_begin + rows_per_split);
  const bool do_bias = bias && blockIdx.y == 0;
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  if (t < 128) bsum[t] = 0.0f;
  if (warp == 0) tmem_alloc(&tslot, 256);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  const int nch = (r_end - r_begin + TNK - 1) / TNK;
  // chunk c: rows r_begin + 32c .. +31; A cols p0..p0+127 (32 float4 per row), B cols
  // q0..q0+Qtp-1; thread t: float4 column group t % 32 (A) of rows t/32 + 8j
  auto convert = [&](int c, int b) {
    const int r0 = r_begin + c * TNK;
    uint8_t* ai = aimg + b * (TNK * 128 * 2);
    uint8_t* bi = bimg + b * (TNK * Qtp * 2);
    float bs[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const int c4 = 4 * (t & 31), p = p0 + c4;
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rl = (t >> 5) + 8 * j, r = r0 + rl;
        v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < r_end) {
          const float* src = A + (int64_t)r * lda + p;
          if (p + 3 < P) v[j] = __ldg(reinterpret_cast<const float4*>(src));
          else {
            if (p < P) v[j].x = __ldg(src);
            if (p + 1 < P) v[j].y = __ldg(src + 1);
            if (p + 2 < P) v[j].z = __ldg(src + 2);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rl = (t >> 5) + 8 * j;
        *reinterpret_cast<uint2*>(ai + (rl >> 3) * (128 * 16) + (c4 >> 3) * 128 + (rl & 7) * 16 +
                                  (c4 & 7) * 2) = make_uint2(pack2(v[j].x, v[j].y), pack2(v[j].z, v[j].w));
        if (do_bias) { bs[0] += v[j].x; bs[1] += v[j].y; bs[2] += v[j].z; bs[3] += v[j].w; }
      }
      if (do_bias) {
        atomicAdd(&bsum[c4], bs[0]); atomicAdd(&bsum[c4 + 1], bs[1]);
        atomicAdd(&bsum[c4 + 2], bs[2]); atomicAdd(&bsum[c4 + 3], bs[3]);
      }
    }
    // B: Qtp/4 float4 groups per row, TNK rows
    const int ng = Qtp / 4;
    for (int e = t; e < ng * TNK; e += 256) {
      const int rl = e / ng, c4 = 4 * (e - rl * ng), r = r0 + rl, q = q0 + c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < r_end && c4 < Qt) {
        const float* src = B + (int64_t)r * ldb + q;
        if (q + 3 < Q && c4 + 3 < Qt) v = __ldg(reinterpret_cast<const float4*>(src));
        else {
          if (q < Q && c4 < Qt) v.x = __ldg(src);
          if (q + 1 < Q && c4 + 1 < Qt) v.y = __ldg(src + 1);
          if (q + 2 < Q && c4 + 2 < Qt) v.z = __ldg(src + 2);
        }
      }
      *reinterpret_cast<uint2*>(bi + (rl >> 3) * (Qtp * 16) + (c4 >> 3) * 128 + (rl & 7) * 16 +
                                (c4 & 7) * 2) = make_uint2(pack2(v.x, v.y), pack2(v.z, v.w));
    }
  };
  const uint32_t idesc = idesc_bf16(128, Qtp, true, true);
  if (nch > 0) {
    convert(0, 0);
    fence_async_smem();
  }
  tc_before();
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int b = c & 1;
    if (t == 0) {
      tc_after();
      gemm(tm, mnmaj(aimg + b * (TNK * 128 * 2), 128), mnmaj(bimg + b * (TNK * Qtp * 2), Qtp), TNK / 16,
           idesc, c > 0);
      mma_commit(&bars[b]);
    }
    if (c + 1 < nch) {
      if (c >= 1) mbar_wait(&bars[b ^ 1], (uint32_t)(((c - 1) >> 1) & 1));
      convert(c + 1, b ^ 1);
      fence_async_smem();
    }
    tc_before();
    __syncthreads();
  }
  if (nch > 0) {
    mbar_wait(&bars[(nch - 1) & 1], (uint32_t)(((nch - 1) >> 1) & 1));
    tc_after();
    // epilogue in column halves of ≤128 through shared memory: TMEM -> tile [128 p][128 q]
    // (lane = p), then warps walk whole p rows, 4 q per lane: the fp32 atomics of a warp
    // hit one contiguous 512-byte row segment
    float* stile = reinterpret_cast<float*>(sm);
    constexpr int LDT = 128 + 4;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_base = tm + ((uint32_t)((warp & 3) * 32) << 16);
    for (int h0 = 0; h0 < Qtp; h0 += 128) {
      const int hn = min(128, Qtp - h0), ngrp = hn / 16, gsplit = (ngrp + 1) / 2;
      const int jb = (warp < 4 ? 0 : gsplit) * 16, je = (warp < 4 ? gsplit : ngrp) * 16;
      for (int jl = jb; jl < je; jl += 16) {
        float v[16];
        tmem_ld16(lane_base + (uint32_t)(h0 + jl), v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(stile + row * LDT + jl + 4 * q) =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      __syncthreads();
      for (int r = warp; r < 128; r += 8) {
        const int p = p0 + r, jl = 4 * lane;
        if (p >= P || jl >= hn) continue;
        const float4 val = *reinterpret_cast<const float4*>(stile + r * LDT + jl);
        const float vv[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int ql = h0 + jl + e, q = q0 + ql;
          if (ql < Qt && q < Q && vv[e] != 0.0f) atomicAdd(C + (int64_t)p * ldc + q, vv[e]);
        }
      }
      __syncthreads();
    }
  }
  tc_before();
  __syncthreads();
  if (do_bias && t < 128 && p0 + t < P && bsum[t] != 0.0f) atomicAdd(bias + p0 + t, bsum[t]);
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 256);
  }
}

// fp32 W_k [w × K_in] -> bf16 image [w rows × Kp cols] (layer k at wimg + off_img[k])
__global__ void k_tc_pack_w(ShArgs a) {
  for (int k = 0; k < a.L; ++k) {
    const int Kin = k == 0 ? a.d + 1 : a.w, Kp = (Kin + 15) / 16 * 16;
    const float* W = a.params + a.off_W[k];
    uint16_t* img = a.wimg + a.off_img[k];
    for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < (int64_t)a.w * Kp;
         id += (int64_t)gridDim.x * blockDim.x) {
      const int r = (int)(id / Kp), c = (int)(id - (int64_t)r * Kp);
      const float x = c < Kin ? W[(int64_t)r * Kin + c] : 0.0f;
      const __nv_bfloat16 h = __float2bfloat16_rn(x);
      const size_t off = (size_t)(r >> 3) * (Kp * 8) + (c >> 3) * 64 + (r & 7) * 8 + (c & 7);
      img[off] = *reinterpret_cast<const uint16_t*>(&h);
    }
  }
}

// out[j] += Σ_r X[r][j] (+ s[r]·Y[r][j]);  blockDim 256 = 8 row lanes × 32 columns
__global__ void __launch_bounds__(NTH) k_colsum(const float* __restrict__ X, int ldx,
                                                const float* __restrict__ s,
                                                const float* __restrict__ Y, int ldy, int R,
                                                int NC, int rows_per_block, float* __restrict__ out) {
  const int j = blockIdx.x * 32 + (threadIdx.x & 31), lr = threadIdx.x >> 5;
  const int r0 = blockIdx.y * rows_per_block, r1 = min(R, r0 + rows_per_block);
  float acc = 0.0f;
  if (j < NC)
    for (int r = r0 + lr; r < r1; r += 8) {
      float v = X ? X[(int64_t)r * ldx + j] : 0.0f;
      if (Y) v = fmaf(s[r], Y[(int64_t)r * ldy + j], v);
      acc += v;
    }
  __shared__ float red[8][33];
  red[lr][threadIdx.x & 31] = acc;
  __syncthreads();
  if (lr == 0 && j < NC) {
    float tot = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += red[k][threadIdx.x & 31];
    if (tot != 0.0f) atomicAdd(out + j, tot);
  }
}

// 128×128 tiles, BK = 8, 8×8 outputs per thread as 2×2 blocks of 4×4 (rows
// 4ty + {0..3} and 64 + 4ty + {0..3}, the same for columns), smem double
// buffer filled from registers one k-step ahead.  Used when the grid has at
// least ~2 waves of such tiles; the 64×64 kernel above covers small problems.
constexpr int BB = 128, BKK = 8;

__device__ __forceinline__ float4 ld4_guard(const float* p, int valid) {
  // 4 consecutive floats, zero beyond `valid` (0..4); p is 16-byte aligned when valid == 4
  if (valid >= 4) return __ldg(reinterpret_cast<const float4*>(p));
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid > 0) v.x = __ldg(p);
  if (valid > 1) v.y = __ldg(p + 1);
  if (valid > 2) v.z = __ldg(p + 2);
  return v;
}

template <class Epi>
__device__ __forceinline__ void mma8x8_epilogue(const float (&acc)[8][8], int i0, int j0, int tx,
                                                int ty, int R, int NC, const Epi& epi) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = i0 + (r < 4 ? 4 * ty + r : 64 + 4 * ty + r - 4);
      const int j = j0 + (c < 4 ? 4 * tx + c : 64 + 4 * tx + c - 4);
      if (i < R && j < NC) epi(i, j, acc[r][c]);
    }
}

// the same with one 4-column call per (row, column group) where the group is whole
template <class Epi>
__device__ __forceinline__ void mma8x8_epilogue_v4(const float (&acc)[8][8], int i0, int j0, int tx,
                                                   int ty, int R, int NC, const Epi& epi) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + (r < 4 ? 4 * ty + r : 64 + 4 * ty + r - 4);
    if (i >= R) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + 64 * h + 4 * tx;
      if (j + 3 < NC) {
        epi.v4(i, j, make_float4(acc[r][4 * h], acc[r][4 * h + 1], acc[r][4 * h + 2], acc[r][4 * h + 3]));
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (j + c < NC) epi(i, j + c, acc[r][4 * h + c]);
      }
    }
  }
}

__device__ __forceinline__ void mma8x8_step(const float (*As)[BB], const float (*Bs)[BB], int tx,
                                            int ty, float (&acc)[8][8]) {
#pragma unroll
  for (int kk = 0; kk < BKK; ++kk) {
    const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][4 * ty]);
    const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][64 + 4 * ty]);
    const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][4 * tx]);
    const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][64 + 4 * tx]);
    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
  }
}

// Row GEMM, big tiles.  A [R×K] row-major with lda % 4 == 0 (all activation
// buffers); B as in k_gemm_rows (any ldb: loaded element-wise, it is a weight
// matrix that stays in L1/L2).
template <bool NT, class Epi>
__global__ void __launch_bounds__(NTH, 2) k_gemm_rows128(const float* __restrict__ A, int lda,
                                                         const float* __restrict__ B, int ldb,
                                                         int R, int NC, int K, Epi epi, Op2 op2) {
  const float* Ap = A;
  const float* Bp = B;
  int ldap = lda, ldbp = ldb, Kp = K;
  __shared__ __align__(16) float As[2][BKK][BB];
  __shared__ __align__(16) float Bs[2][BKK][BB];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int i0 = blockIdx.y * BB, j0 = blockIdx.x * BB;
  // A loads: row t/2, k offset 4(t&1);  B loads: NT row (col j) t/2, k 4(t&1);
  //          NN k = t/32, cols 4(t&31)
  const int ar = t >> 1, ak = 4 * (t & 1);
  float4 ra, rb;
  auto load = [&](int k0) {
    const int i = i0 + ar, k = k0 + ak;
    ra = (i < R) ? ld4_guard(Ap + (int64_t)i * ldap + k, Kp - k) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (NT) {
      const int j = j0 + ar;
      if (j >= NC) {
        rb = make_float4(0.f, 0.f, 0.f, 0.f);
      } else if (ldbp % 4 == 0) {
        rb = ld4_guard(Bp + (int64_t)j * ldbp + k, Kp - k);
      } else {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (k + e < Kp) ? __ldg(Bp + (int64_t)j * ldbp + k + e) : 0.f;
        rb = make_float4(v[0], v[1], v[2], v[3]);
      }
    } else {
      const int kb = k0 + (t >> 5), jb = j0 + 4 * (t & 31);
      if (kb >= Kp) {
        rb = make_float4(0.f, 0.f, 0.f, 0.f);
      } else if (ldbp % 4 == 0) {
        rb = ld4_guard(Bp + (int64_t)kb * ldbp + jb, NC - jb);
      } else {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (jb + e < NC) ? __ldg(Bp + (int64_t)kb * ldbp + jb + e) : 0.f;
        rb = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  };
  auto store = [&](int buf) {
    As[buf][ak + 0][ar] = ra.x; As[buf][ak + 1][ar] = ra.y;
    As[buf][ak + 2][ar] = ra.z; As[buf][ak + 3][ar] = ra.w;
    if (NT) {
      Bs[buf][ak + 0][ar] = rb.x; Bs[buf][ak + 1][ar] = rb.y;
      Bs[buf][ak + 2][ar] = rb.z; Bs[buf][ak + 3][ar] = rb.w;
    } else {
      *reinterpret_cast<float4*>(&Bs[buf][t >> 5][4 * (t & 31)]) = rb;
    }
  };
  float acc[8][8] = {};
  for (int pass = 0; pass < (op2.A ? 2 : 1); ++pass) {
    if (pass) { Ap = op2.A; Bp = op2.B; ldap = op2.lda; ldbp = op2.ldb; Kp = op2.K; }
    load(0);
    store(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < Kp; k0 += BKK) {
      const bool more = k0 + BKK < Kp;
      if (more) load(k0 + BKK);
      mma8x8_step(As[buf], Bs[buf], tx, ty, acc);
      if (more) store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  if (epi.ld % 4 == 0) mma8x8_epilogue_v4(acc, i0, j0, tx, ty, R, NC, epi);
  else mma8x8_epilogue(acc, i0, j0, tx, ty, R, NC, epi);
}

// Weight-gradient GEMM, big tiles: C[p][q] += Σ_r A[r][p]·B[r][q] over this CTA's
// row range, fp32 atomics; bias (optional, blockIdx.x == 0 CTAs): += Σ_r A[r][p].
// lda, ldb % 4 == 0.
__global__ void __launch_bounds__(NTH, 2) k_gemm_tn128(const float* __restrict__ A, int lda,
                                                       const float* __restrict__ B, int ldb, int R,
                                                       int P, int Q, float* __restrict__ C, int ldc,
                                                       float* __restrict__ bias, int rows_per_split) {
  __shared__ __align__(16) float As[2][BKK][BB];
  __shared__ __align__(16) float Bs[2][BKK][BB];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int p0 = blockIdx.y * BB, q0 = blockIdx.x * BB;
  const int r_begin = blockIdx.z * rows_per_split, r_end = min(R, r_begin + rows_per_split);
  const int lk = t >> 5, lc = 4 * (t & 31);
  float4 ra, rb;
  auto load = [&](int r0) {
    const int r = r0 + lk;
    const bool ok = r < r_end;
    ra = ok ? ld4_guard(A + (int64_t)r * lda + p0 + lc, P - p0 - lc) : make_float4(0.f, 0.f, 0.f, 0.f);
    rb = ok ? ld4_guard(B + (int64_t)r * ldb + q0 + lc, Q - q0 - lc) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto store = [&](int buf) {
    *reinterpret_cast<float4*>(&As[buf][lk][lc]) = ra;
    *reinterpret_cast<float4*>(&Bs[buf][lk][lc]) = rb;
  };
  const bool do_bias = bias && blockIdx.x == 0 && t < BB;   // thread t sums column p0 + t
  float acc[8][8] = {};
  float bsum = 0.0f;
  if (r_begin < r_end) {
    load(r_begin);
    store(0);
  }
  __syncthreads();
  int buf = 0;
  for (int r0 = r_begin; r0 < r_end; r0 += BKK) {
    const bool more = r0 + BKK < r_end;
    if (more) load(r0 + BKK);
    mma8x8_step(As[buf], Bs[buf], tx, ty, acc);
    if (do_bias) {
#pragma unroll
      for (int kk = 0; kk < BKK; ++kk) bsum += As[buf][kk][t];
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  struct AtomicEpi {
    float* C;
    int ldc;
    __device__ void operator()(int p, int q, float v) const {
      if (v != 0.0f) atomicAdd(C + (int64_t)p * ldc + q, v);
    }
  };
  mma8x8_epilogue(acc, p0, q0, tx, ty, P, Q, AtomicEpi{C, ldc});
  if (do_bias && p0 + t < P && bsum != 0.0f) atomicAdd(bias + p0 + t, bsum);
}

// out[j] += Σ_r X[r][j] (+ s[r]·Y[r][j]), 4 columns per thread (ldx, ldy % 4 == 0, NC % 4 == 0):
// block = 16 column groups (64 columns) × 16 row lanes
__global__ void __launch_bounds__(NTH) k_colsum4(const float* __restrict__ X, int ldx,
                                                 const float* __restrict__ s,
                                                 const float* __restrict__ Y, int ldy, int R, int NC,
                                                 int rows_per_block, float* __restrict__ out) {
  const int cg = threadIdx.x & 15, lr = threadIdx.x >> 4;
  const int j = blockIdx.x * 64 + 4 * cg;
  const int r0 = blockIdx.y * rows_per_block, r1 = min(R, r0 + rows_per_block);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j < NC)
    for (int r = r0 + lr; r < r1; r += 16) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(X + (int64_t)r * ldx + j));
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      if (Y) {
        const float sv = __ldg(s + r);
        const float4 y = __ldg(reinterpret_cast<const float4*>(Y + (int64_t)r * ldy + j));
        acc.x = fmaf(sv, y.x, acc.x); acc.y = fmaf(sv, y.y, acc.y);
        acc.z = fmaf(sv, y.z, acc.z); acc.w = fmaf(sv, y.w, acc.w);
      }
    }
  __shared__ float4 red[16][17];
  red[lr][cg] = acc;
  __syncthreads();
  if (lr == 0 && j < NC) {
    float4 tot = red[0][cg];
    for (int k = 1; k < 16; ++k) {
      tot.x += red[k][cg].x; tot.y += red[k][cg].y; tot.z += red[k][cg].z; tot.w += red[k][cg].w;
    }
    atomicAdd(out + j, tot.x);
    atomicAdd(out + j + 1, tot.y);
    atomicAdd(out + j + 2, tot.z);
    atomicAdd(out + j + 3, tot.w);
  }
}

// ---------------------------------------------------------------- epilogues
// Each functor has a scalar form and a 4-column form (j % 4 == 0, ld % 4 == 0,
// j + 3 < NC) used by the 128-tile kernels: one 16-byte access per array.
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
#define F4MAP(expr)                                                                  \
  make_float4([&](int e_) { return expr; }(0), [&](int e_) { return expr; }(1),       \
              [&](int e_) { return expr; }(2), [&](int e_) { return expr; }(3))
__device__ __forceinline__ float comp(const float4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

struct EpiFwd {        // layer k: s = tanh(a + b); S_k, H_k (ResNet); δ_L on the last layer
  const float* b;
  float* S;
  float* H;            // != S for ResNet layers k ≥ 2
  const float* Hprev;  // h_{k-1} (ResNet)
  const float* v;      // head (last layer only) for δ_L = v ⊙ (1 - s²)
  float* D;
  int ld;
  __device__ void operator()(int i, int j, float a) const {
    const float s = tanhf(a + __ldg(b + j));
    const int64_t o = (int64_t)i * ld + j;
    S[o] = s;
    if (H != S) H[o] = Hprev[o] + s;
    if (v) D[o] = __ldg(v + j) * (1.0f - s * s);
  }
  __device__ void v4(int i, int j, float4 a) const {
    const int64_t o = (int64_t)i * ld + j;
    const float4 s = F4MAP(tanhf(comp(a, e_) + __ldg(b + j + e_)));
    st4(S + o, s);
    if (H != S) {
      const float4 hp = ld4(Hprev + o);
      st4(H + o, F4MAP(comp(hp, e_) + comp(s, e_)));
    }
    if (v) st4(D + o, F4MAP(__ldg(v + j + e_) * (1.0f - comp(s, e_) * comp(s, e_))));
  }
};

struct EpiIg {         // g_{k-1} = δ_k W_k (+ g_k); δ_{k-1} = g_{k-1} ⊙ (1 - s_{k-1}²)
  const float* gk;     // g_k for the residual term (null: none); gk_is_v: g_L = v (row-broadcast)
  int gk_is_v;
  float* G;            // g_{k-1}
  const float* S;      // s_{k-1} (null for k = 1: g_0 has no δ)
  float* D;            // δ_{k-1}
  int ld;              // of G, S, D (and gk unless gk_is_v)
  __device__ void operator()(int i, int j, float c) const {
    const int64_t o = (int64_t)i * ld + j;
    if (gk) c += gk_is_v ? __ldg(gk + j) : gk[o];
    G[o] = c;
    if (S) {
      const float s = S[o];
      D[o] = c * (1.0f - s * s);
    }
  }
  __device__ void v4(int i, int j, float4 c) const {
    const int64_t o = (int64_t)i * ld + j;
    if (gk) {
      const float4 g = gk_is_v ? F4MAP(__ldg(gk + j + e_)) : ld4(gk + o);
      c = F4MAP(comp(c, e_) + comp(g, e_));
    }
    st4(G + o, c);
    if (S) {
      const float4 s = ld4(S + o);
      st4(D + o, F4MAP(comp(c, e_) * (1.0f - comp(s, e_) * comp(s, e_))));
    }
  }
};

struct EpiUp {         // δ̄_k = ḡ_{k-1} W_kᵀ:  ḡ_k = δ̄ ⊙ s'_k (+ ḡ_{k-1});  s̄_k = -2 s_k g_k δ̄
  const float* S;      // s_k
  const float* Gk;     // g_k (null: g_L = v, row-broadcast from gv)
  const float* gv;
  const float* Gbprev; // ḡ_{k-1} for the residual term (same width w), or null
  float* Gb;           // ḡ_k
  float* Sb;           // s̄_k
  int ld;
  // last layer only: ā_L = (s̄_L + ū v) ⊙ s'_L straight away (and h̄_L = ū v for a
  // residual last layer), instead of storing s̄_L for a separate pass
  const float* ub = nullptr;
  float* Ab = nullptr;
  float* HbL = nullptr;
  __device__ void operator()(int i, int j, float db) const {
    const int64_t o = (int64_t)i * ld + j;
    const float s = S[o];
    const float g = Gk ? Gk[o] : __ldg(gv + j);
    float gb = db * (1.0f - s * s);
    if (Gbprev) gb += Gbprev[o];
    Gb[o] = gb;
    const float sb = -2.0f * s * g * db;
    if (Ab) {
      const float hb = __ldg(ub + i) * __ldg(gv + j);
      if (HbL) HbL[o] = hb;
      Ab[o] = (sb + hb) * (1.0f - s * s);
    } else {
      Sb[o] = sb;
    }
  }
  __device__ void v4(int i, int j, float4 db) const {
    const int64_t o = (int64_t)i * ld + j;
    const float4 s = ld4(S + o);
    const float4 g = Gk ? ld4(Gk + o) : F4MAP(__ldg(gv + j + e_));
    float4 gb = F4MAP(comp(db, e_) * (1.0f - comp(s, e_) * comp(s, e_)));
    if (Gbprev) {
      const float4 gp = ld4(Gbprev + o);
      gb = F4MAP(comp(gb, e_) + comp(gp, e_));
    }
    st4(Gb + o, gb);
    const float4 sb = F4MAP(-2.0f * comp(s, e_) * comp(g, e_) * comp(db, e_));
    if (Ab) {
      const float u = __ldg(ub + i);
      const float4 hb = F4MAP(u * __ldg(gv + j + e_));
      if (HbL) st4(HbL + o, hb);
      st4(Ab + o, F4MAP((comp(sb, e_) + comp(hb, e_)) * (1.0f - comp(s, e_) * comp(s, e_))));
    } else {
      st4(Sb + o, sb);
    }
  }
};

struct EpiDown {       // h̄_{k-1} = ā_k W_k (+ h̄_k);  ā_{k-1} = (s̄_{k-1} + h̄_{k-1}) ⊙ s'_{k-1}
  const float* Hb;     // h̄_k (residual term) or null
  float* Hbout;        // h̄_{k-1} when layer k-1 is itself residual (needed one level down), or null
  const float* Sb;     // s̄_{k-1}
  const float* S;      // s_{k-1}
  float* Ab;           // ā_{k-1}
  int ld;
  __device__ void operator()(int i, int j, float c) const {
    const int64_t o = (int64_t)i * ld + j;
    if (Hb) c += Hb[o];
    if (Hbout) Hbout[o] = c;
    const float s = S[o];
    Ab[o] = (Sb[o] + c) * (1.0f - s * s);
  }
  __device__ void v4(int i, int j, float4 c) const {
    const int64_t o = (int64_t)i * ld + j;
    if (Hb) {
      const float4 h = ld4(Hb + o);
      c = F4MAP(comp(c, e_) + comp(h, e_));
    }
    if (Hbout) st4(Hbout + o, c);
    const float4 s = ld4(S + o), sb = ld4(Sb + o);
    st4(Ab + o, F4MAP((comp(sb, e_) + comp(c, e_)) * (1.0f - comp(s, e_) * comp(s, e_))));
  }
};

// ---------------------------------------------------------------- row kernels
// Paths of this rank: ΔW rows (n·M + m) = ΔW_n and U0 rows (n·M + m) = [t_n, X_n].
// a1 + a2 for the shared formulation, one CTA per path m: (1) the CTA's threads
// draw every (step n, 4-component block q) of the path independently (one Philox
// call per coupled sub-step, R8/R22) and store ΔW_n — the loss and the
// double-backward read it; (2) one thread per component runs the Euler recursion
// over n, its ΔW loads batched 8 steps ahead (the path's rows are L1/L2-hot), and
// writes the rows (t_n, X_n) of U0.  (A thread per (m, q) walking n serially, with
// the draws on the recursion's critical path, took 31 µs at the paper's M = 100.)
__global__ void k_sh_paths(ShArgs a) {
  const int nq = (a.d + 3) >> 2;
  const uint32_t it = a.eval ? a.eval_it : a.state->it;
  const int64_t sdw = a.M * a.d, su = a.M * a.K0p;   // row strides of step n
  for (int64_t m = blockIdx.x; m < a.M; m += gridDim.x) {
    for (int id = threadIdx.x; id < a.N * nq; id += blockDim.x) {
      const int n = id / nq, q = id - n * nq;
      float dw[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < a.cpl; ++j) {
        const float4 z = normals4((uint32_t)q, (uint32_t)(a.m0 + m), (uint32_t)(n * a.cpl + j), it,
                                  a.k0, a.k1);
        dw[0] += a.sqrt_dt_f * z.x; dw[1] += a.sqrt_dt_f * z.y;
        dw[2] += a.sqrt_dt_f * z.z; dw[3] += a.sqrt_dt_f * z.w;
      }
      float* o = a.dW + n * sdw + m * a.d + 4 * q;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < a.d) o[e] = dw[e];
    }
    __syncthreads();   // this path's ΔW rows are visible to the whole CTA
    for (int j = threadIdx.x; j < a.d; j += blockDim.x) {
      const float* dw = a.dW + m * a.d + j;
      float* u = a.U0 + m * a.K0p + 1 + j;
      float x = a.x0;
      int n = 0;
      for (; n + 8 <= a.N; n += 8) {
        float w[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) w[r] = dw[(n + r) * sdw];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          u[(n + r) * su] = x;
          x = x_step(a.problem, x, w[r]);
        }
      }
      for (; n < a.N; ++n) {
        const float w = dw[n * sdw];
        u[n * su] = x;
        x = x_step(a.problem, x, w);
      }
      u[(int64_t)a.N * su] = x;
    }
    for (int n = threadIdx.x; n <= a.N; n += blockDim.x) a.U0[n * su + m * a.K0p] = (float)n * a.dt;
    __syncthreads();
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ∂g/∂x_i given x_i and s = |x|² (R27): heat, Black-Scholes 2x; HJB 2x/(1+s);
// Allen-Cahn -0.8x/(2+0.4s)²
__device__ __forceinline__ float grad_g(int problem, float x, float s) {
  if (problem == kHJB) return 2.0f * x / (1.0f + s);
  if (problem == kAllenCahn) {
    const float q = 2.0f + 0.4f * s;
    return -0.8f * x / (q * q);
  }
  return 2.0f * x;
}

// z_i = σ(X)ᵀ∇ₓu: √2 g_i, or σ x_i g_i (Black-Scholes)
__device__ __forceinline__ float sig(int problem, float x, float g) {
  return problem == kBlackScholes ? kBSSigma * x * g : 1.41421356237309515f * g;
}

// One warp per row: u = v·h_L + c; z·ΔW, |z|², Σz (n < N) or |X_N|² (n = N).
__global__ void k_sh_rowscal(ShArgs a) {
  const int64_t R = (int64_t)(a.N + 1) * a.M;
  const int lane = threadIdx.x & 31;
  const float* v = a.params + a.off_v;
  const float c = a.params[a.off_v + a.w];
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < R;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int n = (int)(r / a.M);
    const float* h = a.HL + r * a.w;
    float u = 0.0f;
    for (int j = lane; j < a.w; j += 32) u = fmaf(h[j], __ldg(v + j), u);
    u = warp_sum(u) + c;
    const float* xr = a.U0 + r * a.K0p + 1;
    const float* gr = a.G0 + r * a.K0p + 1;
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;
    if (n < a.N) {
      const float* dw = a.dW + r * a.d;
      for (int i = lane; i < a.d; i += 32) {
        const float z = sig(a.problem, xr[i], gr[i]);
        s0 = fmaf(z, dw[i], s0);
        s1 = fmaf(z, z, s1);
        s2 += z;
      }
    } else {
      for (int i = lane; i < a.d; i += 32) s0 = fmaf(xr[i], xr[i], s0);
    }
    s0 = warp_sum(s0);
    if (n == a.N && a.zN) {   // Σ_i (∂_i u - ∂_i g)² of the Z_N term (needs |X_N|² = s0)
      for (int i = lane; i < a.d; i += 32) {
        const float e = gr[i] - grad_g(a.problem, xr[i], s0);
        s1 = fmaf(e, e, s1);
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      a.u[r] = u;
      a.q[4 * r + 0] = s0;   // z·ΔW, or |X_N|²
      a.q[4 * r + 1] = s1;   // |z|²
      a.q[4 * r + 2] = s2;   // Σ z
    }
  }
}

__device__ __forceinline__ float residual(const ShArgs& a, int n, int64_t m) {
  const int64_t r = (int64_t)n * a.M + m;
  if (n == a.N) return a.u[r] - terminal_g(a.problem, a.q[4 * r]);
  const float y = a.u[r];
  return a.u[r + a.M] - y + driver_f(a.problem, y, a.q[4 * r + 1], a.q[4 * r + 2], a.lam) * a.dt -
         a.q[4 * r];
}

// One warp per row (n, m): the residuals r_{n-1}, r_n; Σ r²; ū = ∂L/∂u and
// ḡ_0 = [0, σ(X) z̄] with z̄ = (2/B) r_n (Δt ∂_z f - ΔW_n) (R24).
__global__ void k_sh_loss(ShArgs a) {
  const int64_t R = (int64_t)(a.N + 1) * a.M;
  const int lane = threadIdx.x & 31;
  const float sc = 2.0f * a.inv_B;
  const float zc = a.dt * driver_dfdz_coef(a.problem, a.lam), zc0 = a.dt * driver_dfdz_const(a.problem);
  double lsum = 0.0;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < R;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int n = (int)(r / a.M);
    const int64_t m = r - (int64_t)n * a.M;
    const float rn = residual(a, n, m);
    if (lane == 0) lsum += (double)rn * rn;
    if (lane == 0 && n == a.N && a.zN) lsum += (double)a.q[4 * r + 1];   // Z_N term (R27)
    if (a.eval) continue;
    const float y = a.u[r];
    float ub = 0.0f;
    if (n >= 1) ub += residual(a, n - 1, m);
    if (n < a.N) ub += rn * (-1.0f + a.dt * driver_dfdy(a.problem, y));
    else ub += rn;
    float* gb = a.G0b + r * a.K0p;
    if (lane == 0) {
      a.ub[r] = sc * ub;
      gb[0] = 0.0f;
    }
    const float* xr = a.U0 + r * a.K0p + 1;
    if (n < a.N) {
      const float* gr = a.G0 + r * a.K0p + 1;
      const float* dw = a.dW + r * a.d;
      const float f = sc * rn;
      for (int i = lane; i < a.d; i += 32) {
        const float z = sig(a.problem, xr[i], gr[i]);
        gb[1 + i] = sig(a.problem, xr[i], f * (fmaf(zc, z, zc0) - dw[i]));
      }
    } else {
      const float* gr = a.G0 + r * a.K0p + 1;
      const float sN = a.q[4 * r];
      for (int i = lane; i < a.d; i += 32)   // Z_N term: 2/B (∂_i u - ∂_i g), else 0
        gb[1 + i] = a.zN ? sc * (gr[i] - grad_g(a.problem, xr[i], sN)) : 0.0f;
      if (lane == 0) a.Rstore[m] = rn;
    }
  }
  // block reduction of Σ r² (lane 0 of each warp holds a partial)
  __shared__ double red[NTH / 32];
  if (lane == 0) red[threadIdx.x >> 5] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    if (s != 0.0) atomicAdd(a.loss_acc, s);
  }
}

// Y0 = u(0, X_0): one CTA evaluates the network at one point.
__global__ void k_sh_point(ShArgs a, float* out) {
  extern __shared__ float hbuf[];                 // [3][max(K0p, w)]: h, h', u
  const int W = a.w, ldh = a.K0p > W ? a.K0p : W;
  float* h0 = hbuf;
  float* h1 = hbuf + ldh;
  float* u = hbuf + 2 * ldh;
  for (int i = threadIdx.x; i < a.K0p; i += blockDim.x)
    h0[i] = u[i] = (i == 0 || i > a.d) ? 0.0f : a.x0;
  __syncthreads();
  int K = a.d + 1;
  for (int k = 0; k < a.L; ++k) {
    const float* Wk = a.params + a.off_W[k];
    const float* bk = Wk + (int64_t)W * K;
    for (int j = threadIdx.x; j < W; j += blockDim.x) {
      float acc = bk[j];
      if (a.arch == 2 && k > 0) {   // NAIS-Net block: A_k h + B_k u + C_k (A_k from k_sh_nais_A)
        const float* A = a.Am + (int64_t)k * W * W;
        const float* Bk = a.params + a.off_Bk[k];
        for (int i = 0; i < W; ++i) acc = fmaf(A[(int64_t)j * W + i], h0[i], acc);
        for (int i = 0; i <= a.d; ++i) acc = fmaf(Bk[(int64_t)j * (a.d + 1) + i], u[i], acc);
      } else {
        for (int i = 0; i < K; ++i) acc = fmaf(Wk[(int64_t)j * K + i], h0[i], acc);
      }
      const float s = tanhf(acc);
      h1[j] = (a.arch != 0 && k > 0) ? h0[j] + s : s;
    }
    __syncthreads();
    float* tmp = h0; h0 = h1; h1 = tmp;
    K = W;
    __syncthreads();
  }
  float p = 0.0f;
  for (int j = threadIdx.x; j < W; j += blockDim.x) p = fmaf(h0[j], a.params[a.off_v + j], p);
  p = warp_sum(p);
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = a.params[a.off_v + W];
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    *out = s;
  }
}

// NAIS-Net (R26) helpers around the w×w×w products, which run on the GEMM kernels:
// G_k = R_kᵀR_k (weight-gradient GEMM over the w rows of R_k) into the A buffer,
// then A_k = -G_k - εI (k_sh_nais_fix); S_k = Ā_k + Ā_kᵀ (k_sh_nais_sym) and
// R̄_k = -R_k S_k (row GEMM, EpiNeg); ‖G_k‖_F and the projection (k_sh_nais_scale).
__global__ void k_sh_nais_fix(ShArgs a) {
  const int W = a.w;
  const int64_t tot = (int64_t)(a.L - 1) * W * W;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < tot;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(id % ((int64_t)W * W)), i = e / W, j = e - i * W;
    float* A = a.Am + (int64_t)W * W + id;      // blocks k = 1..L-1 start at Am + W·W
    *A = -*A - (i == j ? kNaisEps : 0.0f);
  }
}

__global__ void k_sh_nais_sym(ShArgs a) {      // S_k = Ā_k + Ā_kᵀ from the R_k gradient slot
  const int W = a.w;
  const int64_t tot = (int64_t)(a.L - 1) * W * W;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < tot;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int k = 1 + (int)(id / ((int64_t)W * W));
    const int e = (int)(id - (int64_t)(k - 1) * W * W), i = e / W, j = e - i * W;
    const float* G = a.grad + a.off_W[k];
    a.Am[(int64_t)k * W * W + e] = G[i * W + j] + G[j * W + i];
  }
}

// one CTA per block: f = ‖G_k‖_F (G_k = R_kᵀR_k in the A buffer); R_k *= ((1-ε)/f)^½ if f > 1-ε
__global__ void k_sh_nais_scale(ShArgs a, float* __restrict__ params) {
  const int W = a.w, k = 1 + blockIdx.x;
  const float* Gk = a.Am + (int64_t)k * W * W;
  float* R = params + a.off_W[k];
  double acc = 0.0;
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) acc += (double)Gk[e] * Gk[e];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[32];
  __shared__ float scale;
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double f2 = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) f2 += red[q];
    const double f = sqrt(f2);
    scale = f > 1.0 - kNaisEps ? (float)sqrt((1.0 - kNaisEps) / f) : 1.0f;
  }
  __syncthreads();
  if (scale != 1.0f)
    for (int e = threadIdx.x; e < W * W; e += blockDim.x) R[e] *= scale;
}

__global__ void k_sh_init(float* params, ShArgs a, uint32_t k0, uint32_t k1) {
  // R23: Xavier-uniform W_k (tensor 1 + k), v (tensor 1 + L), zero biases, c ~ U(0,1) (tensor 0)
  const int64_t total = a.off_v + a.w + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t tid = 0, idx = 0;
    int fan_in = 0, fan_out = 0;
    bool weight = false, bias = false;
    if (i >= a.off_v) {
      if (i == a.off_v + a.w) { tid = 0; idx = 0; }
      else { tid = 1 + a.L; idx = (uint32_t)(i - a.off_v); fan_in = a.w; fan_out = 1; weight = true; }
    } else {
      int k = a.L - 1;
      while (i < a.off_W[k]) --k;
      const int K = k == 0 ? a.d + 1 : a.w;
      const int64_t r = i - a.off_W[k];
      if (r < (int64_t)a.w * K) { tid = 1 + k; idx = (uint32_t)r; fan_in = K; fan_out = a.w; weight = true; }
      else if (i >= a.off_Bk[k] && a.arch == 2 && k > 0) {   // NAIS-Net B_k (R26)
        tid = 0x100000u + (uint32_t)k; idx = (uint32_t)(i - a.off_Bk[k]);
        fan_in = a.d + 1; fan_out = a.w; weight = true;
      } else bias = true;
    }
    if (bias) { params[i] = 0.0f; continue; }
    const uint4 x = philox4x32_10(make_uint4(idx >> 2, tid, 0u, kInitStream), k0, k1);
    const uint32_t sel = (idx & 3) == 0 ? x.x : (idx & 3) == 1 ? x.y : (idx & 3) == 2 ? x.z : x.w;
    const float u = unit_from_u32(sel);
    params[i] = weight ? sqrtf(6.0f / (float)(fan_in + fan_out)) * (2.0f * u - 1.0f) : u;
  }
}

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

template <bool NT, class Epi>
cudaError_t gemm_rows(const float* A, int lda, const float* B, int ldb, int R, int NC, int K,
                      const Epi& epi, cudaStream_t s, Op2 op2 = Op2{}) {
  const int64_t big_tiles = (int64_t)((NC + BB - 1) / BB) * ((R + BB - 1) / BB);
  if (lda % 4 == 0 && (!op2.A || op2.lda % 4 == 0) && big_tiles >= 2 * 148) {
    dim3 grid((NC + BB - 1) / BB, (R + BB - 1) / BB);
    k_gemm_rows128<NT, Epi><<<grid, NTH, 0, s>>>(A, lda, B, ldb, R, NC, K, epi, op2);
  } else {
    dim3 grid((NC + TB - 1) / TB, (R + TB - 1) / TB);
    k_gemm_rows<NT, Epi><<<grid, NTH, 0, s>>>(A, lda, B, ldb, R, NC, K, epi, op2);
  }
  return cudaGetLastError();
}

// tcgen05 row GEMM with layer k's bf16 image (NT: N = w, K = K_in; NN: K = w, N = K_in)
template <bool NT, class Epi>
cudaError_t tc_rows(const ShArgs& a, int k, const float* A, int lda, int R, int K, int NC,
                    const Epi& epi, cudaStream_t s) {
  const int Kin = k == 0 ? a.d + 1 : a.w, Kp = (Kin + 15) / 16 * 16;
  const int Npad = NT ? (a.w + 15) / 16 * 16 : Kp;
  constexpr int TN = TCN;   // (TCN/2 at the paper's R = 5 100, 160 CTAs instead of 80: measured slower)
  // weight slab: NT [TN rows × Kp], NN [w rows × TN]
  size_t smem = 2 * 128 * TCK * 2 + (size_t)TN * (NT ? Kp : a.w) * 2;
  const size_t stage = (size_t)128 * (TN + 4) * sizeof(float);   // the epilogue tile
  if (smem < stage) smem = stage;
  RET(cudaFuncSetAttribute(k_tc_rowgemm<NT, Epi, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem));
  dim3 grid((Npad + TN - 1) / TN, (R + 127) / 128);
  k_tc_rowgemm<NT, Epi, TN><<<grid, 256, smem, s>>>(A, lda, R, K, a.wimg + a.off_img[k], a.w, Kp,
                                                     NC, Npad, epi);
  return cudaGetLastError();
}

// C[P×Q] += Aᵀ B over R rows (+ bias[p] += Σ_r A[r][p] when bias != null)
cudaError_t gemm_tn(const float* A, int lda, const float* B, int ldb, int R, int P, int Q, float* C,
                    int ldc, float* bias, cudaStream_t s) {
  const int tiles = ((P + BB - 1) / BB) * ((Q + BB - 1) / BB);
  // CTA target: one per SM for short reductions (the paper's R = 5 100: 296 and 592
  // measured 4-8% slower), two per SM for long ones (R = 2e5: 3% faster)
#ifndef BSDE_EXP_TNS_CTAS
#define BSDE_EXP_TNS_CTAS (R < 32768 ? 148 : 296)
#endif
#ifndef BSDE_EXP_TNS_MINROWS
#define BSDE_EXP_TNS_MINROWS (8 * BKK)
#endif
  int splits = (BSDE_EXP_TNS_CTAS + tiles - 1) / tiles;
  const int max_splits = (R + BSDE_EXP_TNS_MINROWS - 1) / (BSDE_EXP_TNS_MINROWS);   // rows per split
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  int rows = (R + splits - 1) / splits;
  rows = (rows + BKK - 1) / BKK * BKK;
  splits = (R + rows - 1) / rows;
  dim3 grid((Q + BB - 1) / BB, (P + BB - 1) / BB, splits);
  k_gemm_tn128<<<grid, NTH, 0, s>>>(A, lda, B, ldb, R, P, Q, C, ldc, bias, rows);
  return cudaGetLastError();
}

// bf16 tcgen05 weight-gradient GEMM (precision BF16 of the shared formulation)
cudaError_t gemm_tn_tc(const float* A, int lda, const float* B, int ldb, int R, int P, int Q,
                       float* C, int ldc, float* bias, cudaStream_t s) {
  const int Qt = Q <= 256 ? Q : 256;
  const int Qtp = (Qt + 15) / 16 * 16;
  const int tiles = ((P + 127) / 128) * ((Q + Qt - 1) / Qt);
#ifndef BSDE_EXP_TN_CTAS
#define BSDE_EXP_TN_CTAS 296
#endif
  int splits = (BSDE_EXP_TN_CTAS + tiles - 1) / tiles;
#ifndef BSDE_EXP_TCTN_MINROWS
#define BSDE_EXP_TCTN_MINROWS (4 * TNK)
#endif
  const int max_splits = (R + BSDE_EXP_TCTN_MINROWS - 1) / (BSDE_EXP_TCTN_MINROWS);   // rows per split
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  int rows = (R + splits - 1) / splits;
  rows = (rows + TNK - 1) / TNK * TNK;
  splits = (R + rows - 1) / rows;
  size_t smem = 2 * (size_t)TNK * 128 * 2 + 2 * (size_t)TNK * Qtp * 2;
  if (smem < (size_t)128 * 132 * sizeof(float)) smem = (size_t)128 * 132 * sizeof(float);   // epilogue tile
  RET(cudaFuncSetAttribute(k_tc_tngemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((P + 127) / 128, (Q + Qt - 1) / Qt, splits);
  k_tc_tngemm<<<grid, 256, smem, s>>>(A, lda, B, ldb, R, P, Q, C, ldc, bias, rows, Qt);
  return cudaGetLastError();
}

cudaError_t colsum(const float* X, int ldx, const float* sv, const float* Y, int ldy, int R, int NC,
                   float* out, cudaStream_t s) {
  if (NC % 4 == 0 && ldx % 4 == 0 && (!Y || ldy % 4 == 0)) {
    const int cb = (NC + 63) / 64;
    int rb = (4 * 148 + cb - 1) / cb;
    int rows = (R + rb - 1) / rb;
    if (rows < 64) rows = 64;
    rb = (R + rows - 1) / rows;
    k_colsum4<<<dim3(cb, rb), NTH, 0, s>>>(X, ldx, sv, Y, ldy, R, NC, rows, out);
    return cudaGetLastError();
  }
  const int cb = (NC + 31) / 32;
  int rb = (2 * 148 + cb - 1) / cb;
  int rows = (R + rb - 1) / rb;
  if (rows < 64) rows = 64;
  rb = (R + rows - 1) / rows;
  k_colsum<<<dim3(cb, rb), NTH, 0, s>>>(X, ldx, sv, Y, ldy, R, NC, rows, out);
  return cudaGetLastError();
}

struct EpiNeg {        // out = -c (R̄_k = -R_k S_k)
  float* out;
  int ld;
  __device__ void operator()(int i, int j, float c) const { out[(int64_t)i * ld + j] = -c; }
  __device__ void v4(int i, int j, float4 c) const {
    *reinterpret_cast<float4*>(out + (int64_t)i * ld + j) = make_float4(-c.x, -c.y, -c.z, -c.w);
  }
};



// G_k = R_kᵀR_k for the NAIS-Net blocks into the A buffer (TN GEMM over R's rows)
cudaError_t nais_gram(const ShArgs& a, const float* params, cudaStream_t s) {
  const int W = a.w;
  RET(cudaMemsetAsync(a.Am + (int64_t)W * W, 0, sizeof(float) * (size_t)(a.L - 1) * W * W, s));
  for (int k = 1; k < a.L; ++k) {
    const float* R = params + a.off_W[k];
    RET(gemm_tn(R, W, R, W, W, W, W, a.Am + (int64_t)k * W * W, W, nullptr, s));
  }
  return cudaSuccess;
}

}  // namespace

size_t shared_num_params(int d, int w, int L, int arch) {
  const size_t blk = (size_t)w * w + w + (arch == 2 ? (size_t)w * (d + 1) : 0);
  return (size_t)w * (d + 1) + w + (size_t)(L - 1) * blk + w + 1;
}

void shared_offsets(ShArgs& a) {
  int64_t off = 0;
  for (int k = 0; k < a.L; ++k) {
    a.off_W[k] = off;
    const int K = k == 0 ? a.d + 1 : a.w;
    off += (int64_t)a.w * K + a.w;
    a.off_Bk[k] = off;
    if (a.arch == 2 && k > 0) off += (int64_t)a.w * (a.d + 1);   // B_k after R_k, C_k
  }
  a.off_v = off;
}

// Device buffers for R_max = (N_max + 1)·M rows.
size_t shared_buffer_bytes(int d, int w, int L, int arch, int N_max, int64_t M) {
  const int64_t R = (int64_t)(N_max + 1) * M;
  const int K0p = (d + 1 + 3) & ~3;
  size_t f = 0;
  f += (size_t)R * K0p * 3;                 // U0, G0, G0b
  f += (size_t)N_max * M * d;               // ΔW
  f += (size_t)R * w * (size_t)L * 2;       // S_k, δ_k
  f += (size_t)R * w * (size_t)(L - 1);     // g_1..g_{L-1}
  if (arch != 0) f += (size_t)R * w * (size_t)(L - 1);   // H_k, k ≥ 2
  f += (size_t)R * w * (size_t)L;           // s̄_k
  f += (size_t)R * w * 4;                   // ḡ ping-pong, ā ping-pong
  if (arch != 0) f += (size_t)R * w * 2;    // h̄ ping-pong
  f += (size_t)R * 6;                       // u, ū, q[4]
  if (arch == 2) f += (size_t)L * w * w;    // A_k
  f += ((size_t)w * ((d + 1 + 15) / 16 * 16) + (size_t)(L - 1) * w * ((w + 15) / 16 * 16) + 1) / 2;
  return f * sizeof(float) + 256 * 80;
}

void shared_carve(ShArgs& a, void* base, int N_max) {
  const int64_t R = (int64_t)(N_max + 1) * a.M;
  float* p = static_cast<float*>(base);
  auto take = [&](size_t n) { float* q = p; p += (n + 63) & ~(size_t)63; return q; };
  a.U0 = take((size_t)R * a.K0p);
  a.G0 = take((size_t)R * a.K0p);
  a.G0b = take((size_t)R * a.K0p);
  a.dW = take((size_t)N_max * a.M * a.d);
  for (int k = 0; k < a.L; ++k) {
    a.S[k] = take((size_t)R * a.w);
    a.D[k] = take((size_t)R * a.w);
    a.Sb[k] = take((size_t)R * a.w);
    a.G[k] = k < a.L - 1 ? take((size_t)R * a.w) : nullptr;
    a.H[k] = (a.arch != 0 && k > 0) ? take((size_t)R * a.w) : a.S[k];
  }
  a.HL = a.H[a.L - 1];
  a.Gb[0] = take((size_t)R * a.w);
  a.Gb[1] = take((size_t)R * a.w);
  a.Ab[0] = take((size_t)R * a.w);
  a.Ab[1] = take((size_t)R * a.w);
  if (a.arch != 0) {
    a.Hb[0] = take((size_t)R * a.w);
    a.Hb[1] = take((size_t)R * a.w);
  } else {
    a.Hb[0] = a.Hb[1] = nullptr;
  }
  a.u = take((size_t)R);
  a.ub = take((size_t)R);
  a.q = take((size_t)R * 4);
  a.Am = a.arch == 2 ? take((size_t)a.L * a.w * a.w) : nullptr;
  int64_t img = 0;   // bf16 weight images (tcgen05 row GEMMs)
  for (int k = 0; k < a.L; ++k) {
    a.off_img[k] = img;
    img += (int64_t)a.w * (((k == 0 ? a.d + 1 : a.w) + 15) / 16 * 16);
  }
  a.wimg = reinterpret_cast<uint16_t*>(take((size_t)(img + 1) / 2));
}

cudaError_t launch_shared_init(float* params, const ShArgs& a, uint32_t k0, uint32_t k1,
                               cudaStream_t s) {
  k_sh_init<<<grid_for(a.off_v + a.w + 1, NTH), NTH, 0, s>>>(params, a, k0, k1);
  RET(cudaGetLastError());
  return a.arch == 2 ? launch_shared_nais_project(a, params, s) : cudaSuccess;   // R26
}

cudaError_t launch_shared_nais_project(const ShArgs& a, float* params, cudaStream_t s) {
  if (a.arch != 2 || a.L < 2) return cudaSuccess;
  RET(nais_gram(a, params, s));
  k_sh_nais_scale<<<a.L - 1, NTH, 0, s>>>(a, params);
  return cudaGetLastError();
}

cudaError_t launch_shared_point(const ShArgs& a, float* out, cudaStream_t s) {
  const int ldh = a.K0p > a.w ? a.K0p : a.w;
  if (a.arch == 2) {
    RET(nais_gram(a, a.params, s));
    k_sh_nais_fix<<<grid_for((int64_t)(a.L - 1) * a.w * a.w, NTH), NTH, 0, s>>>(a);
    RET(cudaGetLastError());
  }
  k_sh_point<<<1, 256, 3 * ldh * sizeof(float), s>>>(a, out);
  return cudaGetLastError();
}

// One iteration's forward, loss and (unless a.eval) gradient into a.grad.
// mid (optional) is recorded between the loss and the double-backward pass.
// Returns the number of kernels launched in *launches.
cudaError_t launch_shared_step(const ShArgs& a, cudaStream_t s, cudaEvent_t mid, int* launches) {
  const int R = (a.N + 1) * (int)a.M;
  const int W = a.w, K0 = a.d + 1, L = a.L;
  const bool nais = a.arch == 2;
  const bool res = a.arch == 1 || nais;      // NAIS-Net blocks are residual with h = 1 (R26)
  const bool tcg = a.tc && !nais;            // bf16 tcgen05 row GEMMs
  // weight gradients on tcgen05 too once the row reduction is long enough to hide the
  // fp32 -> bf16 staging (measured at R = 5 100: 1.6% faster per iteration than the
  // SIMT kernel with its one-CTA-per-SM split; faster at 2e5)
#ifndef BSDE_EXP_TCTN_MINR
#define BSDE_EXP_TCTN_MINR 4096
#endif
  const bool tctn = tcg && R >= BSDE_EXP_TCTN_MINR;
  const float* P = a.params;
  int nl = 0;
  // the layer matrix of the forward/back-propagation GEMMs: W_k, or A_k for a NAIS block
  auto Wk = [&](int k) { return (nais && k > 0) ? a.Am + (int64_t)k * W * W : P + a.off_W[k]; };
  auto Bk = [&](int k) { return P + a.off_Bk[k]; };
  auto bk = [&](int k) { return P + a.off_W[k] + (int64_t)W * (k == 0 ? K0 : W); };
  const float* v = P + a.off_v;
  // paths
  k_sh_paths<<<(unsigned)(a.M < 65536 ? a.M : 65536), 128, 0, s>>>(a);
  RET(cudaGetLastError());
  ++nl;
  if (tcg) {    // bf16 images of this iteration's W_k
    k_tc_pack_w<<<grid_for((int64_t)W * W, NTH), NTH, 0, s>>>(a);
    RET(cudaGetLastError());
    ++nl;
  }
  if (nais) {   // A_k = -R_kᵀR_k - εI from this iteration's parameters
    RET(nais_gram(a, a.params, s));
    k_sh_nais_fix<<<grid_for((int64_t)(L - 1) * W * W, NTH), NTH, 0, s>>>(a);
    RET(cudaGetLastError());
    nl += L;
  }
  // forward: layers 1..L (0-based k); NAIS-Net blocks add the input injection u B_kᵀ
  for (int k = 0; k < L; ++k) {
    EpiFwd e{bk(k), a.S[k], a.H[k], k > 0 ? a.H[k - 1] : nullptr, k == L - 1 ? v : nullptr,
             a.D[L - 1], W};
    const float* A = k == 0 ? a.U0 : a.H[k - 1];
    const int lda = k == 0 ? a.K0p : W, K = k == 0 ? K0 : W;
    Op2 inj;
    if (nais && k > 0) inj = Op2{a.U0, a.K0p, Bk(k), K0, K0};
    if (tcg) RET(tc_rows<true>(a, k, A, lda, R, K, W, e, s));
    else RET(gemm_rows<true>(A, lda, Wk(k), K, R, W, K, e, s, inj));
    ++nl;
  }
  // input gradient: g_{k-1} = δ_k W_k (+ g_k), k = L..2, then g_0 = δ_1 W_1; NAIS-Net
  // blocks also add δ_k B_k to g_0 (the first such term initialises g_0)
  bool g0_init = false;
  for (int k = L - 1; k >= 1; --k) {
    const float* gk = res ? (k == L - 1 ? v : a.G[k]) : nullptr;
    EpiIg e{gk, (res && k == L - 1) ? 1 : 0, a.G[k - 1], a.S[k - 1], a.D[k - 1], W};
    if (tcg) RET(tc_rows<false>(a, k, a.D[k], W, R, W, W, e, s));
    else RET(gemm_rows<false>(a.D[k], W, Wk(k), W, R, W, W, e, s));
    ++nl;
    if (nais) {
      EpiIg eu{g0_init ? a.G0 : nullptr, 0, a.G0, nullptr, nullptr, a.K0p};
      RET(gemm_rows<false>(a.D[k], W, Bk(k), K0, R, K0, W, eu, s));
      ++nl;
      g0_init = true;
    }
  }
  {
    EpiIg e{g0_init ? a.G0 : nullptr, 0, a.G0, nullptr, nullptr, a.K0p};
    if (tcg) RET(tc_rows<false>(a, 0, a.D[0], W, R, W, K0, e, s));
    else RET(gemm_rows<false>(a.D[0], W, Wk(0), K0, R, K0, W, e, s));
    ++nl;
  }
  // per-row scalars and the loss
  k_sh_rowscal<<<grid_for((int64_t)R * 32, NTH), NTH, 0, s>>>(a);
  RET(cudaGetLastError());
  k_sh_loss<<<grid_for((int64_t)R * 32, NTH), NTH, 0, s>>>(a);
  RET(cudaGetLastError());
  nl += 2;
  if (mid) cudaEventRecord(mid, s);
  if (a.eval) { if (launches) *launches = nl; return cudaSuccess; }
  float* G = a.grad;
  auto gW = [&](int k) { return G + a.off_W[k]; };
  auto gb = [&](int k) { return G + a.off_W[k] + (int64_t)W * (k == 0 ? K0 : W); };
  float* gv = G + a.off_v;
  // up: k = 1..L (0-based 0..L-1): W̄_k += δ_kᵀ ḡ_{k-1}; δ̄_k = ḡ_{k-1} W_kᵀ -> ḡ_k, s̄_k
  const float* gprev = a.G0b;
  int ldprev = a.K0p;
  for (int k = 0; k < L; ++k) {
    const int K = k == 0 ? K0 : W;
    // W̄_k (NAIS-Net: Ā_k, transformed to R̄_k at the end) += δ_kᵀ ḡ_{k-1}
    if (tctn) RET(gemm_tn_tc(a.D[k], W, gprev, ldprev, R, W, K, gW(k), K, nullptr, s));
    else RET(gemm_tn(a.D[k], W, gprev, ldprev, R, W, K, gW(k), K, nullptr, s));
    Op2 inj;
    if (nais && k > 0) {   // B̄_k += δ_kᵀ ḡ_u;  δ̄_k += ḡ_u B_kᵀ
      RET(gemm_tn(a.D[k], W, a.G0b, a.K0p, R, W, K0, G + a.off_Bk[k], K0, nullptr, s));
      ++nl;
      inj = Op2{a.G0b, a.K0p, Bk(k), K0, K0};
    }
    float* gout = a.Gb[k & 1];
    EpiUp e{a.S[k], k < L - 1 ? a.G[k] : nullptr, v, (res && k > 0) ? gprev : nullptr, gout,
            a.Sb[k], W};
    if (k == L - 1) {   // fuse ā_L (former k_sh_abar_last) into the last up-product
      e.ub = a.ub;
      e.Ab = a.Ab[0];
      e.HbL = res ? a.Hb[0] : nullptr;
    }
    if (tcg) RET(tc_rows<true>(a, k, gprev, ldprev, R, K, W, e, s));
    else RET(gemm_rows<true>(gprev, ldprev, Wk(k), K, R, W, K, e, s, inj));
    nl += 2;
    gprev = gout;
    ldprev = W;
  }
  // head: v̄ = Σ (ḡ_L + ū h_L), c̄ = Σ ū
  RET(colsum(gprev, W, a.ub, a.HL, W, R, W, gv, s));
  RET(colsum(a.ub, 1, nullptr, nullptr, 0, R, 1, gv + W, s));
  nl += 2;
  // down: ā_L, then k = L..1: W̄_k += ā_kᵀ h_{k-1}, b̄_k += Σ ā_k, ā_{k-1} = (s̄_{k-1} + ā_k W_k (+ h̄_k)) ⊙ s'
  int cur = 0;
  // ā_L (and h̄_L) were written by the last up-product's epilogue into Ab[0] / Hb[0]
  for (int k = L - 1; k >= 0; --k) {
    const float* hin = k == 0 ? a.U0 : a.H[k - 1];
    const int K = k == 0 ? K0 : W, ldh = k == 0 ? a.K0p : W;
    if (nais && k > 0) {   // Ā_k += ā_kᵀ h_{k-1};  B̄_k += ā_kᵀ u, C̄_k += Σ ā_k
      RET(gemm_tn(a.Ab[cur], W, hin, ldh, R, W, K, gW(k), K, nullptr, s));
      RET(gemm_tn(a.Ab[cur], W, a.U0, a.K0p, R, W, K0, G + a.off_Bk[k], K0, gb(k), s));
      nl += 2;
    } else {
      if (tctn) RET(gemm_tn_tc(a.Ab[cur], W, hin, ldh, R, W, K, gW(k), K, gb(k), s));
      else RET(gemm_tn(a.Ab[cur], W, hin, ldh, R, W, K, gW(k), K, gb(k), s));   // + b̄_k = Σ ā_k
      ++nl;
    }
    if (k == 0) break;
    const int nxt = cur ^ 1;
    EpiDown e{(res && k > 0) ? a.Hb[cur] : nullptr, (res && k - 1 > 0) ? a.Hb[nxt] : nullptr,
              a.Sb[k - 1], a.S[k - 1], a.Ab[nxt], W};
    if (tcg) RET(tc_rows<false>(a, k, a.Ab[cur], W, R, W, W, e, s));
    else RET(gemm_rows<false>(a.Ab[cur], W, Wk(k), W, R, W, W, e, s));
    ++nl;
    cur = nxt;
  }
  if (nais) {   // R̄_k = -R_k(Ā_k + Ā_kᵀ) (A_k is no longer needed: its buffer holds S_k)
    k_sh_nais_sym<<<grid_for((int64_t)(L - 1) * W * W, NTH), NTH, 0, s>>>(a);
    RET(cudaGetLastError());
    for (int k = 1; k < L; ++k)
      RET(gemm_rows<false>(P + a.off_W[k], W, a.Am + (int64_t)k * W * W, W, W, W, W,
                           EpiNeg{G + a.off_W[k], W}, s));
    nl += L;
  }
  if (launches) *launches = nl;
  return cudaSuccess;
}

}  // namespace bsde
