// rows_tc.cu — the per-step nets at fp32-accurate precision on tcgen05 (BSDE_FP32 with
// kernel TC: configs 1, 2, 4, DESIGN R18b).
//
// bf16x3: a GEMM operand x is split into hi = bf16(x) and lo = bf16(x - hi), and every
// product is accumulated as three bf16 MMAs hi·hi + hi·lo + lo·hi in fp32 TMEM: the
// relative error of a product is ~2^-16, far below the 1e-4 parity tolerance and two
// orders above fp32 rounding only where a ReLU mask is decided (R18b, kink band 2e-5).
//
// X does not depend on θ, so once the paths are drawn every (step n, path m) pair is an
// independent row, and the iteration is a short chain of launches over R = N·B rows,
// grouped over the steps (blockIdx.y / .z = n picks step n's weights):
//   paths  ΔW_n (Philox4x32-10 + MUFU Box-Muller, R8) and the Euler
//          states X_{n+1} = X_n + √2 ΔW_n (Eq. 5) of every row: X̃ = [X, 1, 0..]
//   F1     A1 = X̃ W̃1ᵀ,  H1 = ReLU(A1)                       (Eq. 7; R4)
//   F2     A2 = H1 W̃2ᵀ,  H2 = H1 + ReLU(A2)
//   F3     Z = H2 W̃3ᵀ; per row Z·ΔW and |Z|² (HJB) or Σ Z (Black-Scholes), and
//          G = ΔW - Δt ∂_z f (the factor of ā in dZ) in place of ΔW
//   Y      per path: Y_{n+1} = Y_n - f Δt + Z·ΔW (Eq. 5, R2), R = Y_N - g(X_N), the loss
//          (Eq. 6 terminal term), ā_N (times P_N), dY0
//   B1     dH2 = dZ W̃3 with dZ = ā_{n+1} G formed while staging the operand
//   B2     dH1 = dH2 + dA2 W̃2, dA2 = dH2 ⊙ 1[A2 > 0] staged; dA1 = dH1 ⊙ 1[A1 > 0]
//   TN     dW̃1 = Σ_m dA1ᵀ X̃, dW̃2 = Σ_m dA2ᵀ H1, dW̃3 = Σ_m dZᵀ H2 (the constant-1
//          columns give the bias gradients), split over row ranges, fp32 atomics
// The biases are folded into the weight images (column d of W̃1, column w of W̃2, W̃3;
// W̃1 row w = e_d makes H1[w] = H2[w] = 1), as in the bf16 kernels (tc.cu).
// Row buffers are fp32 [N][B][Dp | Wp] (Dp = pad16(d+1), Wp = pad16(w+1)).
#include <cuda_fp16.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace bsde {
namespace rows {

using namespace tc;

constexpr int RT = 256;   // threads of the GEMM kernels

__host__ __device__ inline uint32_t img_bytes(int r, int c) { return (uint32_t)r * c * 2; }

// bf16 hi / lo of four fp32 values, as two bf16x2 words each
__device__ __forceinline__ void split4(float4 v, uint2& hi, uint2& lo) {
  const __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y), h1 = __floats2bfloat162_rn(v.z, v.w);
  const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
  const __nv_bfloat162 l0 = __floats2bfloat162_rn(v.x - f0.x, v.y - f0.y);
  const __nv_bfloat162 l1 = __floats2bfloat162_rn(v.z - f1.x, v.w - f1.y);
  hi = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
  lo = make_uint2(*reinterpret_cast<const uint32_t*>(&l0), *reinterpret_cast<const uint32_t*>(&l1));
}
// byte offset of (r, c) (c % 4 == 0: 8 bytes) in an [R × C] operand image (tc_common.cuh)
__device__ __forceinline__ uint32_t ioff(int r, int c, int C) {
  return (uint32_t)((r >> 3) * (C * 16) + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}

// ------------------------------------------------------------------ weight images
// per step n: [W̃1 hi | W̃2 hi | W̃3 hi | W̃1 lo | W̃2 lo | W̃3 lo] (tc.cu k_pack_tc layout)
__global__ void k_rows_pack(RowsArgs a, int N) {
  const int d = a.d, w = a.w, Dp = a.Dp, Wp = a.Wp;
  const NetDims nd{d, w};
  const int c1 = Wp * (Dp / 4), c2 = Wp * (Wp / 4), c3 = Dp * (Wp / 4);   // float4 groups
  const int per = c1 + c2 + c3;
  const uint32_t WB = img_bytes(Wp, Dp) + img_bytes(Wp, Wp) + img_bytes(Dp, Wp);
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < (int64_t)N * per;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(id / per);
    int r = (int)(id - (int64_t)n * per);
    const float* P = a.params + nd.step_base(n);
    uint8_t* img = a.wimg_w + (size_t)n * 2 * WB;
    int row, c4, C;
    float v[4];
    if (r < c1) {                       // W̃1 [Wp × Dp]: [W1 | b1], row w = e_d
      C = Dp; row = r / (C / 4); c4 = 4 * (r - row * (C / 4));
      for (int e = 0; e < 4; ++e) {
        const int k = c4 + e;
        float x = 0.0f;
        if (row < w) x = k < d ? P[nd.off_W1() + row * d + k] : (k == d ? P[nd.off_b1() + row] : 0.0f);
        else if (row == w) x = k == d ? 1.0f : 0.0f;
        v[e] = x;
      }
    } else if (r < c1 + c2) {           // W̃2 [Wp × Wp]: [W2 | b2]
      r -= c1; img += img_bytes(Wp, Dp);
      C = Wp; row = r / (C / 4); c4 = 4 * (r - row * (C / 4));
      for (int e = 0; e < 4; ++e) {
        const int k = c4 + e;
        v[e] = row < w ? (k < w ? P[nd.off_W2() + row * w + k] : (k == w ? P[nd.off_b2() + row] : 0.0f))
                       : 0.0f;
      }
    } else {                            // W̃3 [Dp × Wp]: [W3 | b3]
      r -= c1 + c2; img += img_bytes(Wp, Dp) + img_bytes(Wp, Wp);
      C = Wp; row = r / (C / 4); c4 = 4 * (r - row * (C / 4));
      for (int e = 0; e < 4; ++e) {
        const int k = c4 + e;
        v[e] = row < d ? (k < w ? P[nd.off_W3() + row * w + k] : (k == w ? P[nd.off_b3() + row] : 0.0f))
                       : 0.0f;
      }
    }
    uint2 hi, lo;
    split4(make_float4(v[0], v[1], v[2], v[3]), hi, lo);
    *reinterpret_cast<uint2*>(img + ioff(row, c4, C)) = hi;
    *reinterpret_cast<uint2*>(img + WB + ioff(row, c4, C)) = lo;
  }
}

// ------------------------------------------------------------------ paths
// one warp per path, lane q = columns 4q..4q+3 (Dp <= 128)
__global__ void __launch_bounds__(256) k_rows_paths(RowsArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t m = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (m >= a.B) return;
  const int d = a.d, Dp = a.Dp, q = lane;
  const bool live = 4 * q < Dp, gen = 4 * q < d;
  const uint32_t it = a.eval ? a.eval_it : a.state->it;
  const uint32_t mg = (uint32_t)(a.m0 + m);
  const bool mult = a.problem == kBlackScholes;
  float X[4];
  for (int e = 0; e < 4; ++e) X[e] = a.x0;
  for (int n = 0; n < a.N; ++n) {
    float dw[4] = {0.f, 0.f, 0.f, 0.f};
    if (gen) {
      for (int j = 0; j < a.cpl; ++j) {   // coupled paths: the sum of the fine increments
        // the MUFU Box-Muller of the tensor-core kernels (R8; ~1e-6 relative, pinned by
        // test_fast_normals_match_oracle), four times the rate of the libm map
        const float4 z = dw4_fast((uint32_t)q, mg, (uint32_t)(n * a.cpl + j), it, a.k0, a.k1,
                                  a.sqrt_dt_f);
        dw[0] += z.x; dw[1] += z.y; dw[2] += z.z; dw[3] += z.w;
      }
    }
    if (live) {
      float xv[4], gv[4];
      for (int e = 0; e < 4; ++e) {
        const int c = 4 * q + e;
        xv[e] = c < d ? X[e] : (c == d ? 1.0f : 0.0f);
        gv[e] = c < d ? dw[e] : 0.0f;
      }
      const size_t o = ((size_t)n * a.B + m) * Dp + 4 * q;
      *reinterpret_cast<float4*>(a.XT + o) = make_float4(xv[0], xv[1], xv[2], xv[3]);
      *reinterpret_cast<float4*>(a.GW + o) = make_float4(gv[0], gv[1], gv[2], gv[3]);
    }
    for (int e = 0; e < 4; ++e)
      if (4 * q + e < d) X[e] = mult ? fmaf(kBSSigma * dw[e], X[e], X[e]) : fmaf(1.41421356237309515f, dw[e], X[e]);
  }
  float s = 0.0f;
  for (int e = 0; e < 4; ++e)
    if (4 * q + e < d) s = fmaf(X[e], X[e], s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) a.xn2[m] = s;
}

// ------------------------------------------------------------------ row GEMMs
enum { F1 = 0, F2 = 1, F3 = 2, B1 = 3, B2 = 4 };

// ā_{n+1} of row (n, m): ā_N P_N / P_{n+1} (per_step_abar problems) or ā_N
__device__ __forceinline__ float abar_of(const RowsArgs& a, int n, int64_t m) {
  const float ab = a.abar[m];
  return per_step_abar(a.problem) ? __fdividef(ab, a.Pstore[(int64_t)n * a.B + m]) : ab;
}

// One CTA per (row-tile group, step n): step n's weight images are loaded once, then
// the CTA walks its 128-row tiles (tile = blockIdx.x, + gridDim.x, ...): stage the A
// tile as bf16 hi / lo images, three MMA passes, fused epilogue out of TMEM.  Two
// CTAs fit an SM (smem sized to the operands), so one stages while the other multiplies.
template <int OP>
__global__ void __launch_bounds__(RT, 2) k_rows_gemm(RowsArgs a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tslot;
  __shared__ float sred[2][2][128];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int n = blockIdx.y;
  const int Dp = a.Dp, Wp = a.Wp, d = a.d;
  // K (A columns) and Nc (output columns); the weight image and its use
  const int K = (OP == F1 || OP == B1) ? Dp : Wp;
  const int Nc = (OP == F3) ? Dp : Wp;
  const int mat = (OP == F1) ? 0 : (OP == F2 || OP == B2) ? 1 : 2;   // W̃1, W̃2, W̃3
  constexpr bool NN = OP == B1 || OP == B2;                           // A·W̃ (else A·W̃ᵀ)
  const uint32_t WB = img_bytes(Wp, Dp) + img_bytes(Wp, Wp) + img_bytes(Dp, Wp);
  const uint32_t moff = mat == 0 ? 0u : mat == 1 ? img_bytes(Wp, Dp) : img_bytes(Wp, Dp) + img_bytes(Wp, Wp);
  const uint32_t mbytes = img_bytes(Nc, K);
  uint8_t* whi = sm;
  uint8_t* wlo = sm + mbytes;
  uint8_t* ahi = sm + 2 * mbytes;
  uint8_t* alo = ahi + img_bytes(128, K);
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 128);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  if (t == 0) {   // step n's weight images, hi and lo
    const uint8_t* src = a.wimg + (size_t)n * 2 * WB + moff;
    mbar_expect_tx(&bars[0], 2 * mbytes);
    for (uint32_t o = 0; o < mbytes; o += 16384u) {
      bulk_g2s(whi + o, src + o, min(16384u, mbytes - o), &bars[0]);
      bulk_g2s(wlo + o, src + WB + o, min(16384u, mbytes - o), &bars[0]);
    }
  }
  const uint32_t idesc = idesc_bf16(128, Nc, false, NN);
  const int ntiles = (int)((a.B + 127) / 128);
  const int q = warp & 3, h = warp >> 2, rr = 32 * q + lane;
  const uint32_t lb = tm + ((uint32_t)(32 * q) << 16);
  const int cb = h * (Nc / 2), nch8 = Nc / 16;   // this warp's 8-column chunks: cb + 8j, j < nch8
  const float dt = a.dt;
  uint32_t ph = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ph ^= 1) {
    const int64_t i0 = (int64_t)tile * 128;
    // stage A (fp32 -> bf16 hi / lo images [128 × K]): float4 groups, coalesced per row,
    // SU groups per thread with all their loads in flight before any conversion
    const int g4 = K / 4;
    constexpr int SU = (OP == B2) ? 2 : 4;
    for (int e0 = t; e0 < 128 * g4; e0 += RT * SU) {
      float4 vv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
      const int e = e0 + u * RT;
      const int r = e / g4, c = 4 * (e - r * g4);
      const int64_t m = i0 + r;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < 128 * g4 && m < a.B) {
        const size_t row = (size_t)n * a.B + m;
        if (OP == F1) v = __ldg(reinterpret_cast<const float4*>(a.XT + row * Dp + c));
        if (OP == F2) v = __ldg(reinterpret_cast<const float4*>(a.H1 + row * Wp + c));
        if (OP == F3) v = __ldg(reinterpret_cast<const float4*>(a.H2 + row * Wp + c));
        if (OP == B1) {   // dZ = ā_{n+1} G (columns >= d of G are 0)
          const float ab = abar_of(a, n, m);
          const float4 gv = __ldg(reinterpret_cast<const float4*>(a.GW + row * Dp + c));
          v = make_float4(ab * gv.x, ab * gv.y, ab * gv.z, ab * gv.w);
        }
        if (OP == B2) {   // dA2 = dH2 ⊙ 1[A2 > 0], A2 > 0 <=> H2 > H1 (R15)
          const float4 g = __ldg(reinterpret_cast<const float4*>(a.DH + row * Wp + c));
          const float4 h1 = __ldg(reinterpret_cast<const float4*>(a.H1 + row * Wp + c));
          const float4 h2 = __ldg(reinterpret_cast<const float4*>(a.H2 + row * Wp + c));
          v = make_float4(h2.x > h1.x ? g.x : 0.f, h2.y > h1.y ? g.y : 0.f, h2.z > h1.z ? g.z : 0.f,
                          h2.w > h1.w ? g.w : 0.f);
        }
      }
      vv[u] = v;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int e = e0 + u * RT;
        if (e >= 128 * g4) break;
        const int r = e / g4, c = 4 * (e - r * g4);
        uint2 hi, lo;
        split4(vv[u], hi, lo);
        *reinterpret_cast<uint2*>(ahi + ioff(r, c, K)) = hi;
        *reinterpret_cast<uint2*>(alo + ioff(r, c, K)) = lo;
      }
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (t == 0) {
      tc_after();
      if (tile == (int)blockIdx.x) mbar_wait(&bars[0], 0);
      const Opnd Ah = kmaj(ahi, K), Al = kmaj(alo, K);
      const Opnd Wh = NN ? mnmaj(whi, Nc) : kmaj(whi, K), Wl = NN ? mnmaj(wlo, Nc) : kmaj(wlo, K);
      gemm(tm, Ah, Wh, K / 16, idesc, false);
      gemm(tm, Ah, Wl, K / 16, idesc, true);
      gemm(tm, Al, Wh, K / 16, idesc, true);
      mma_commit(&bars[1]);
    }
    mbar_wait(&bars[1], ph);
    tc_after();
    // epilogue: warp (q, h) = lanes 32q.., columns [h·Nc/2, (h+1)·Nc/2), all loads in flight
    const int64_t m = i0 + rr;
    const bool ok = m < a.B;
    const size_t row = (size_t)n * a.B + (ok ? m : 0);
    float s1 = 0.f, s2 = 0.f;
    uint32_t r8[8][8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nch8) tmem_ld8_nowait(lb + (uint32_t)(cb + 8 * j), r8[j]);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j >= nch8) break;
      reg_fence8(r8[j]);
      if (!ok) continue;
      const int c0 = cb + 8 * j;
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r8[j][e]);
      if (OP == F1) {
        float* dst = a.H1 + row * Wp + c0;
        *reinterpret_cast<float4*>(dst) = make_float4(fmaxf(v[0], 0.f), fmaxf(v[1], 0.f), fmaxf(v[2], 0.f), fmaxf(v[3], 0.f));
        *reinterpret_cast<float4*>(dst + 4) = make_float4(fmaxf(v[4], 0.f), fmaxf(v[5], 0.f), fmaxf(v[6], 0.f), fmaxf(v[7], 0.f));
      }
      if (OP == F2) {
        const float4 p0 = *reinterpret_cast<const float4*>(a.H1 + row * Wp + c0);
        const float4 p1 = *reinterpret_cast<const float4*>(a.H1 + row * Wp + c0 + 4);
        float* dst = a.H2 + row * Wp + c0;
        *reinterpret_cast<float4*>(dst) = make_float4(p0.x + fmaxf(v[0], 0.f), p0.y + fmaxf(v[1], 0.f),
                                                      p0.z + fmaxf(v[2], 0.f), p0.w + fmaxf(v[3], 0.f));
        *reinterpret_cast<float4*>(dst + 4) = make_float4(p1.x + fmaxf(v[4], 0.f), p1.y + fmaxf(v[5], 0.f),
                                                          p1.z + fmaxf(v[6], 0.f), p1.w + fmaxf(v[7], 0.f));
      }
      if (OP == F3) {   // Z·ΔW, |Z|² | Σ Z; G = ΔW - Δt ∂_z f in place (R2)
        float* gp = a.GW + row * Dp + c0;
        float g[8];
        *reinterpret_cast<float4*>(g) = *reinterpret_cast<const float4*>(gp);
        *reinterpret_cast<float4*>(g + 4) = *reinterpret_cast<const float4*>(gp + 4);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (c0 + e >= d) { g[e] = 0.f; continue; }
          s1 = fmaf(v[e], g[e], s1);
          if (a.problem == kHJB) s2 = fmaf(v[e], v[e], s2);
          else if (a.problem == kBlackScholes) s2 += v[e];
          // ∂_z f = -λ z (HJB), r/σ (Black-Scholes), 0 (heat, Allen-Cahn)
          g[e] = fmaf(-dt, driver_dfdz_coef(a.problem, a.lam) * v[e] + driver_dfdz_const(a.problem), g[e]);
        }
        if (!a.eval) {
          *reinterpret_cast<float4*>(gp) = *reinterpret_cast<const float4*>(g);
          *reinterpret_cast<float4*>(gp + 4) = *reinterpret_cast<const float4*>(g + 4);
        }
      }
      if (OP == B1) {
        float* dst = a.DH + row * Wp + c0;
        *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
      }
      if (OP == B2) {   // dH1 = dH2 + dA2 W̃2; dA1 = dH1 ⊙ 1[A1 > 0] = 1[H1 > 0]
        float dh[8], h1[8];
        *reinterpret_cast<float4*>(dh) = *reinterpret_cast<const float4*>(a.DH + row * Wp + c0);
        *reinterpret_cast<float4*>(dh + 4) = *reinterpret_cast<const float4*>(a.DH + row * Wp + c0 + 4);
        *reinterpret_cast<float4*>(h1) = *reinterpret_cast<const float4*>(a.H1 + row * Wp + c0);
        *reinterpret_cast<float4*>(h1 + 4) = *reinterpret_cast<const float4*>(a.H1 + row * Wp + c0 + 4);
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = h1[e] > 0.f ? dh[e] + v[e] : 0.f;
        *reinterpret_cast<float4*>(a.DA + row * Wp + c0) = *reinterpret_cast<const float4*>(o);
        *reinterpret_cast<float4*>(a.DA + row * Wp + c0 + 4) = *reinterpret_cast<const float4*>(o + 4);
      }
    }
    if (OP == F3) {   // the two column halves of a row
      sred[0][h][rr] = s1;
      sred[1][h][rr] = s2;
    }
    tc_before();
    __syncthreads();   // TMEM read and the A images consumed: the next tile may overwrite them
    if (OP == F3 && h == 0 && ok)
      *reinterpret_cast<float2*>(a.S + row * 2) = make_float2(sred[0][0][rr] + sred[0][1][rr],
                                                             sred[1][0][rr] + sred[1][1][rr]);
    if (OP == F3) __syncthreads();   // sred read before the next tile writes it
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 128);
  }
}

// ------------------------------------------------------------------ Y recursion, loss, ā
__global__ void __launch_bounds__(256) k_rows_y(RowsArgs a) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  __shared__ double lred[8];
  __shared__ float gred[8];
  double l = 0.0;
  float g0 = 0.0f;
  if (m < a.B) {
    float Y = a.params[0], P = 1.0f;
    const bool pa = per_step_abar(a.problem) && !a.eval;
    for (int n = 0; n < a.N; ++n) {
      const float2 s = *reinterpret_cast<const float2*>(a.S + ((size_t)n * a.B + m) * 2);
      if (pa) {
        P *= 1.0f - a.dt * driver_dfdy(a.problem, Y);
        a.Pstore[(int64_t)n * a.B + m] = P;
      }
      Y = Y - driver_f(a.problem, Y, s.y, s.y, a.lam) * a.dt + s.x;
    }
    const float R = Y - terminal_g(a.problem, a.xn2[m]);
    l = (double)R * R;
    if (!a.eval) {
      a.Rstore[m] = R;
      float ab = 2.0f * R * a.inv_B;
      if (per_step_abar(a.problem)) ab *= P;
      a.abar[m] = ab;
      g0 = ab;
    }
  }
  for (int o = 16; o; o >>= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
    g0 += __shfl_xor_sync(0xffffffffu, g0, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { lred[warp] = l; gred[warp] = g0; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double L = 0.0;
    float G0 = 0.0f;
    for (int k = 0; k < 8; ++k) { L += lred[k]; G0 += gred[k]; }
    if (L != 0.0) atomicAdd(a.loss_acc, L);
    if (!a.eval && G0 != 0.0f) atomicAdd(a.grad, G0);
  }
}

// ------------------------------------------------------------------ weight gradients
// blockIdx.y = which: 0 dW̃1 = Σ dA1ᵀ X̃, 1 dW̃2 = Σ dA2ᵀ H1, 2 dW̃3 = Σ dZᵀ H2 over the rows
// [r0, r1) of step n = blockIdx.z; M = 128 (output rows p < P), N = Q, K = 32 rows a chunk
constexpr int TK = 32;
__global__ void __launch_bounds__(RT) k_rows_tn(RowsArgs a, int rows_per_cta) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int which = blockIdx.y, n = blockIdx.z;
  const int Dp = a.Dp, Wp = a.Wp, d = a.d, w = a.w;
  const int P = which == 2 ? Dp : Wp, Q = which == 0 ? Dp : Wp;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta, r1 = (a.B < r0 + rows_per_cta ? a.B : r0 + rows_per_cta);
  // per buffer: A hi, A lo [TK × 128], B hi, B lo [TK × Q]
  const uint32_t AB = img_bytes(TK, 128), BB = img_bytes(TK, Q), BUF = 2 * AB + 2 * BB;
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 128);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  const int nch = r0 < r1 ? (int)((r1 - r0 + TK - 1) / TK) : 0;
  auto convert = [&](int c, int b) {
    uint8_t* base = sm + b * BUF;
    const int64_t rb = r0 + (int64_t)c * TK;
    // A: [TK rows × 128 cols] (columns >= P zero); all of a thread's loads in flight first
    constexpr int UA = TK * 32 / RT;
    float4 va[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int e = t + u * RT;
      const int rl = e >> 5, c4 = 4 * (e & 31);
      const int64_t m = rb + rl;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < r1 && c4 < P) {
        const size_t row = (size_t)n * a.B + m;
        if (which == 0) v = __ldg(reinterpret_cast<const float4*>(a.DA + row * Wp + c4));
        if (which == 1) {
          const float4 g = __ldg(reinterpret_cast<const float4*>(a.DH + row * Wp + c4));
          const float4 h1 = __ldg(reinterpret_cast<const float4*>(a.H1 + row * Wp + c4));
          const float4 h2 = __ldg(reinterpret_cast<const float4*>(a.H2 + row * Wp + c4));
          v = make_float4(h2.x > h1.x ? g.x : 0.f, h2.y > h1.y ? g.y : 0.f, h2.z > h1.z ? g.z : 0.f,
                          h2.w > h1.w ? g.w : 0.f);
        }
        if (which == 2) {
          const float ab = abar_of(a, n, m);
          const float4 gv = __ldg(reinterpret_cast<const float4*>(a.GW + row * Dp + c4));
          v = make_float4(ab * gv.x, ab * gv.y, ab * gv.z, ab * gv.w);
        }
      }
      va[u] = v;
    }
    // B loads of the chunk, then all conversions
    const int q4 = Q / 4;
    constexpr int UB = (TK * 32 + RT - 1) / RT;   // Q <= 128: at most TK·32 groups
    float4 vb[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int e = t + u * RT;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < TK * q4) {
        const int rl = e / q4, c4 = 4 * (e - rl * q4);
        const int64_t m = rb + rl;
        if (m < r1) {
          const size_t row = (size_t)n * a.B + m;
          if (which == 0) v = __ldg(reinterpret_cast<const float4*>(a.XT + row * Dp + c4));
          if (which == 1) v = __ldg(reinterpret_cast<const float4*>(a.H1 + row * Wp + c4));
          if (which == 2) v = __ldg(reinterpret_cast<const float4*>(a.H2 + row * Wp + c4));
        }
      }
      vb[u] = v;
    }
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int e = t + u * RT;
      const int rl = e >> 5, c4 = 4 * (e & 31);
      uint2 hi, lo;
      split4(va[u], hi, lo);
      *reinterpret_cast<uint2*>(base + ioff(rl, c4, 128)) = hi;
      *reinterpret_cast<uint2*>(base + AB + ioff(rl, c4, 128)) = lo;
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int e = t + u * RT;
      if (e >= TK * q4) break;
      const int rl = e / q4, c4 = 4 * (e - rl * q4);
      uint2 hi, lo;
      split4(vb[u], hi, lo);
      *reinterpret_cast<uint2*>(base + 2 * AB + ioff(rl, c4, Q)) = hi;
      *reinterpret_cast<uint2*>(base + 2 * AB + BB + ioff(rl, c4, Q)) = lo;
    }
  };
  const uint32_t idesc = idesc_bf16(128, Q, true, true);
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
      uint8_t* base = sm + b * BUF;
      const Opnd Ah = mnmaj(base, 128), Al = mnmaj(base + AB, 128);
      const Opnd Bh = mnmaj(base + 2 * AB, Q), Bl = mnmaj(base + 2 * AB + BB, Q);
      gemm(tm, Ah, Bh, TK / 16, idesc, c > 0);
      gemm(tm, Ah, Bl, TK / 16, idesc, true);
      gemm(tm, Al, Bh, TK / 16, idesc, true);
      mma_commit(&bars[b]);
    }
    if (c + 1 < nch) {
      if (c >= 1) mbar_wait(&bars[b ^ 1], (uint32_t)(((c - 1) >> 1) & 1));   // chunk c-1 read it
      convert(c + 1, b ^ 1);
      fence_async_smem();
    }
    tc_before();
    __syncthreads();
  }
  if (nch > 0) {
    mbar_wait(&bars[(nch - 1) & 1], (uint32_t)(((nch - 1) >> 1) & 1));
    tc_after();
    // accumulator lane p = output row, columns q: the flat gradient of step n
    const NetDims nd{d, w};
    float* G = a.grad + nd.step_base(n);
    const int qd = warp & 3, hh = warp >> 2, p = 32 * qd + lane;
    const uint32_t lb = tm + ((uint32_t)(32 * qd) << 16);
    const int cb = hh * (Q / 2), ce = cb + Q / 2;
    for (int c0 = cb; c0 < ce; c0 += 8) {
      uint32_t r8[8];
      tmem_ld8_nowait(lb + (uint32_t)c0, r8);
      tmem_ld_wait();
      reg_fence8(r8);
      for (int e = 0; e < 8; ++e) {
        const int k = c0 + e;
        const float v = __uint_as_float(r8[e]);
        if (v == 0.0f) continue;
        int64_t off = -1;
        if (which == 0 && p < w) off = k < d ? nd.off_W1() + p * d + k : (k == d ? nd.off_b1() + p : -1);
        if (which == 1 && p < w) off = k < w ? nd.off_W2() + p * w + k : (k == w ? nd.off_b2() + p : -1);
        if (which == 2 && p < d) off = k < w ? nd.off_W3() + p * w + k : (k == w ? nd.off_b3() + p : -1);
        if (off >= 0) atomicAdd(G + off, v);
      }
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 128);
  }
}

inline int pad16(int x) { return (x + 15) / 16 * 16; }
inline int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}
template <int OP>
cudaError_t gemm_launch(const RowsArgs& a, cudaStream_t s) {
  const int K = (OP == F1 || OP == B1) ? a.Dp : a.Wp, Nc = (OP == F3) ? a.Dp : a.Wp;
  const size_t smem = 2 * (size_t)img_bytes(Nc, K) + 2 * (size_t)img_bytes(128, K);
  cudaError_t e = cudaFuncSetAttribute(k_rows_gemm<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  // two CTAs per SM over the N steps; each walks the row tiles of its step
  const int ntiles = (int)((a.B + 127) / 128), sms = sm_count();
  int g = (2 * sms + a.N - 1) / a.N;
  if (g > ntiles) g = ntiles;
  if (g < 1) g = 1;
  k_rows_gemm<OP><<<dim3((unsigned)g, (unsigned)a.N), RT, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rows

bool rows_supported(int d, int w) { return d + 1 <= 128 && w + 1 <= 128; }

size_t rows_buffer_bytes(int d, int w, int N, int64_t B) {
  const size_t Dp = rows::pad16(d + 1), Wp = rows::pad16(w + 1), R = (size_t)N * B;
  return 4 * (2 * R * Dp + 4 * R * Wp + 2 * R + B) + 6 * 256;
}
size_t rows_pack_bytes(int d, int w, int N) {
  const int Dp = rows::pad16(d + 1), Wp = rows::pad16(w + 1);
  return (size_t)N * 2 * (rows::img_bytes(Wp, Dp) + rows::img_bytes(Wp, Wp) + rows::img_bytes(Dp, Wp));
}

// carve the row buffers [N_max][B] from base (rows_buffer_bytes)
void rows_carve(RowsArgs& a, void* base, int N_max) {
  a.Dp = rows::pad16(a.d + 1);
  a.Wp = rows::pad16(a.w + 1);
  uint8_t* p = static_cast<uint8_t*>(base);
  const size_t R = (size_t)N_max * a.B;
  auto take = [&](size_t floats) {
    float* f = reinterpret_cast<float*>(p);
    p += (floats * 4 + 255) / 256 * 256;
    return f;
  };
  a.XT = take(R * a.Dp);
  a.GW = take(R * a.Dp);
  a.H1 = take(R * a.Wp);
  a.H2 = take(R * a.Wp);
  a.DH = take(R * a.Wp);
  a.DA = take(R * a.Wp);
  a.S = take(R * 2);
  a.xn2 = take(a.B);
}

cudaError_t launch_rows_pack(const RowsArgs& a, cudaStream_t s) {
  const int per = a.Wp * (a.Dp / 4) + a.Wp * (a.Wp / 4) + a.Dp * (a.Wp / 4);
  const int64_t total = (int64_t)a.N * per;
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  rows::k_rows_pack<<<grid, 256, 0, s>>>(a, a.N);
  return cudaGetLastError();
}

#define RCK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

// forward: paths, F1-F3, Y (a.eval: forward only, nothing for the adjoint is kept)
cudaError_t launch_rows_forward(const RowsArgs& a, cudaStream_t s, int* launches) {
  rows::k_rows_paths<<<(unsigned)((a.B * 32 + 255) / 256), 256, 0, s>>>(a);
  RCK(cudaGetLastError());
  RCK(rows::gemm_launch<rows::F1>(a, s));
  RCK(rows::gemm_launch<rows::F2>(a, s));
  RCK(rows::gemm_launch<rows::F3>(a, s));
  rows::k_rows_y<<<(unsigned)((a.B + 255) / 256), 256, 0, s>>>(a);
  RCK(cudaGetLastError());
  if (launches) *launches += 5;
  return cudaSuccess;
}

// adjoint: B1, B2 and the three weight-gradient GEMMs (one launch)
cudaError_t launch_rows_backward(const RowsArgs& a, cudaStream_t s, int* launches) {
  RCK(rows::gemm_launch<rows::B1>(a, s));
  RCK(rows::gemm_launch<rows::B2>(a, s));
  // about four CTAs per SM over the 3·N weight-gradient problems, >= 256 rows each
  const int sms = rows::sm_count();
  int split = (int)((4LL * sms + 3LL * a.N - 1) / (3LL * a.N));
  const int64_t maxsplit = (a.B + 255) / 256;
  if (split > maxsplit) split = (int)maxsplit;
  if (split < 1) split = 1;
  const int rpc = (int)((a.B + split - 1) / split);
  const int Qmax = a.Dp > a.Wp ? a.Dp : a.Wp;
  const size_t smem = 2 * (2 * (size_t)rows::img_bytes(rows::TK, 128) + 2 * (size_t)rows::img_bytes(rows::TK, Qmax));
  RCK(cudaFuncSetAttribute(rows::k_rows_tn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  rows::k_rows_tn<<<dim3((unsigned)((a.B + rpc - 1) / rpc), 3, (unsigned)a.N), rows::RT, smem, s>>>(a, rpc);
  RCK(cudaGetLastError());
  if (launches) *launches += 3;
  return cudaSuccess;
}

}  // namespace bsde
