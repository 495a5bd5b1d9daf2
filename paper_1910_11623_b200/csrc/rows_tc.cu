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
//   B1     dH2 = dZ W̃3 with dZ = ā_{n+1} G formed while staging the operand;
//          dA2 = dH2 ⊙ 1[A2 > 0]
//   B2     dH1 = dH2 + dA2 W̃2, dA1 = dH1 ⊙ 1[A1 > 0]
// For the built shapes F1 + F2 and B1 + B2 are fused kernels (k_rows_f12_t,
// k_rows_b12_t): the masks 1[A1 > 0], 1[A2 > 0] are taken from the accumulators and
// stored as bit words; the unfused B1 / B2 (runtime shapes) test H2 > H1 and H1 > 0,
// which equal them except where ReLU(A2) is below half an ulp of H1.
//   TN     dW̃1 = Σ_m dA1ᵀ X̃, dW̃2 = Σ_m dA2ᵀ H1, dW̃3 = Σ_m dZᵀ H2 (the constant-1
//          columns give the bias gradients), fp32 atomics per (which, step) segment
// The biases are folded into the weight images (column d of W̃1, column w of W̃2, W̃3;
// W̃1 row w = e_d makes H1[w] = H2[w] = 1), as in the bf16 kernels (tc.cu).
// Row buffers are [N][Bs][Dp | Wp] (Dp = pad16(d+1), Wp = pad16(w+1)).  Runtime shapes
// keep fp32 rows (Bs = B).  The built shapes (BSDE_ROWS_SHAPES) keep the buffers that
// only feed GEMM operands — X̃, H1, H2, dA2, dA1 and dZ = ā G — as bf16 hi / lo tile
// images (Bs = B rounded up to 128-row tiles; see "tile images" below), so that the
// weight gradients (k_rows_tn_img) and F3 stream them into the MMAs without
// converting; the launch sequence there is paths, F12, F3, Y | B12, TN.
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

// float4 slot e of a row-major [R × C] fp32 tile -> (row r, column c): each warp's
// 32 slots cover 8 consecutive rows × 16 columns, so the 8-byte stores of its bf16
// halves fill two whole 128-byte core-matrix blocks of the operand image (no bank
// conflicts; a row-major walk puts 16 lanes on the same banks)
template <int C>
__device__ __forceinline__ void slot_rc(int e, int& r, int& c) {
  constexpr int NCG = C / 16;
  const int wi = e >> 5, l = e & 31;
  const int rg = wi / NCG, cg = wi - rg * NCG;
  r = 8 * rg + (l & 7);
  c = 16 * cg + 4 * (l >> 3);
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
// Thread (path m, column quad q < Dp/4): paths packed back to back, Dp/4 threads each
// (blocks of PPB whole paths), so every lane of a warp draws or stores and a warp's
// 16-byte row stores are one contiguous run; |X_N|² summed over a path's threads in
// shared memory, in column order (deterministic).
constexpr int PPB = 8;   // paths per block
__global__ void __launch_bounds__(PPB * 32) k_rows_paths(RowsArgs a) {
  __shared__ float sq[PPB][32];
  const int Q4 = a.Dp / 4;
  const int lp = threadIdx.x / Q4, q = threadIdx.x - lp * Q4;
  const int64_t m = (int64_t)blockIdx.x * PPB + lp;
  const bool act = lp < PPB && m < a.B;
  const int d = a.d, Dp = a.Dp;
  const bool gen = act && 4 * q < d;
  const uint32_t it = a.eval ? a.eval_it : a.state->it;
  const uint32_t mg = (uint32_t)(a.m0 + m);
  const bool mult = a.problem == kBlackScholes;
  float X[4];
  for (int e = 0; e < 4; ++e) X[e] = a.x0;
  if (act) {
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
      float xv[4], gv[4];
      for (int e = 0; e < 4; ++e) {
        const int c = 4 * q + e;
        xv[e] = c < d ? X[e] : (c == d ? 1.0f : 0.0f);
        gv[e] = c < d ? dw[e] : 0.0f;
      }
      const size_t o = ((size_t)n * a.Bs + m) * Dp + 4 * q;
      *reinterpret_cast<float4*>(a.XT + o) = make_float4(xv[0], xv[1], xv[2], xv[3]);
      *reinterpret_cast<float4*>(a.GW + o) = make_float4(gv[0], gv[1], gv[2], gv[3]);
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < d) X[e] = mult ? fmaf(kBSSigma * dw[e], X[e], X[e]) : fmaf(1.41421356237309515f, dw[e], X[e]);
    }
    float s2 = 0.0f;
    for (int e = 0; e < 4; ++e)
      if (4 * q + e < d) s2 = fmaf(X[e], X[e], s2);
    sq[lp][q] = s2;
  }
  __syncthreads();
  if (threadIdx.x < PPB) {
    const int64_t mm = (int64_t)blockIdx.x * PPB + threadIdx.x;
    if (mm < a.B) {
      float s = 0.0f;
      for (int k = 0; k < Q4; ++k) s += sq[threadIdx.x][k];
      a.xn2[mm] = s;
    }
  }
}

// ------------------------------------------------------------------ tile images
// Compile-time shapes keep the row buffers that only feed GEMM operands as bf16 hi / lo
// operand images, per (step n, 128-row tile): [hi 128×C | lo 128×C] in the core-matrix
// layout ioff(r, c, C) (tc_common.cuh), the bytes of the fp32 rows they replace.  The
// same bytes are a K-major A operand of a 128-row tile (F3 reads H2 so) and, half a
// tile at a time, an MN-major operand over 64 rows (the weight-gradient kernel), so no
// consumer converts anything.  X̃, H1, H2, dA1, dA2 and dZ = ā G are images; ΔW / G
// stays fp32 rows (F3 rewrites it, B12 scales it).  Rows past B are zero in every image.
__device__ __forceinline__ uint8_t* tile_img(const float* buf, const RowsArgs& a, int n, int64_t i0, int C) {
  return reinterpret_cast<uint8_t*>(const_cast<float*>(buf) + ((size_t)n * a.Bs + (size_t)i0) * C);
}

// ------------------------------------------------------------------ row GEMMs
enum { F1 = 0, F2 = 1, F3 = 2, B1 = 3, B2 = 4 };

// ā_{n+1} of row (n, m): ā_N P_N / P_{n+1} (per_step_abar problems) or ā_N
__device__ __forceinline__ float abar_of(const RowsArgs& a, int n, int64_t m) {
  const float ab = a.abar[m];
  return per_step_abar(a.problem) ? __fdividef(ab, a.Pstore[(int64_t)n * a.B + m]) : ab;
}

// One CTA per SM-share of step n's row tiles (tile = blockIdx.x, + gridDim.x, ...):
// step n's weight images are loaded once; the fp32 source tile (128 consecutive rows
// of a [N][B][K] buffer: one contiguous block) arrives by bulk copy, is converted to
// bf16 hi / lo images, and the next tile's copy is issued at once, so it lands while
// this tile is multiplied (three MMA passes) and written out.  The epilogue runs in
// two phases through shared memory: TMEM -> a padded [128 × Nc] tile (lane = row),
// then each warp walks whole rows, four columns per lane, so every global access of
// the fused elementwise work is a coalesced row segment.
// Sources: F1 X̃, F2 H1, F3 H2, B1 G (scaled by ā_{n+1} while converting), B2 dA2.
template <int OP>
__global__ void __launch_bounds__(RT, 1) k_rows_gemm(RowsArgs a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[3];   // weights, MMA, raw tile
  __shared__ uint32_t tslot;
  __shared__ float srow[128];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int n = blockIdx.y;
  const int Dp = a.Dp, Wp = a.Wp, d = a.d;
  const int K = (OP == F1 || OP == B1) ? Dp : Wp;    // A columns = source row stride
  const int Nc = (OP == F3) ? Dp : Wp;
  const int ldt = Nc + 4;                            // padded tile row (conflict-free phase 1)
  const int mat = (OP == F1) ? 0 : (OP == F2 || OP == B2) ? 1 : 2;   // W̃1, W̃2, W̃3
  constexpr bool NN = OP == B1 || OP == B2;                           // A·W̃ (else A·W̃ᵀ)
  const float* src = OP == F1 ? a.XT : OP == F2 ? a.H1 : OP == F3 ? a.H2 : OP == B1 ? a.GW : a.DH;
  const uint32_t WB = img_bytes(Wp, Dp) + img_bytes(Wp, Wp) + img_bytes(Dp, Wp);
  const uint32_t moff = mat == 0 ? 0u : mat == 1 ? img_bytes(Wp, Dp) : img_bytes(Wp, Dp) + img_bytes(Wp, Wp);
  const uint32_t mbytes = img_bytes(Nc, K), abytes = img_bytes(128, K);
  uint8_t* whi = sm;
  uint8_t* wlo = sm + mbytes;
  uint8_t* ahi = sm + 2 * mbytes;
  uint8_t* alo = ahi + abytes;
  float* rawt = reinterpret_cast<float*>(alo + abytes);   // [128 × K]
  float* stile = rawt + 128 * K;                           // [128 × ldt]
  const int ntiles = (int)((a.B + 127) / 128);
  auto prefetch = [&](int tile) {   // thread 0: rows of `tile` -> rawt
    const int64_t i0 = (int64_t)tile * 128;
    const uint32_t rows = (uint32_t)(a.B - i0 < 128 ? a.B - i0 : 128);
    const uint32_t bytes = rows * K * 4u;
    const uint8_t* g = reinterpret_cast<const uint8_t*>(src + ((size_t)n * a.Bs + i0) * K);
    uint8_t* dst = reinterpret_cast<uint8_t*>(rawt);
    mbar_expect_tx(&bars[2], bytes);
    for (uint32_t o = 0; o < bytes; o += 16384u) bulk_g2s(dst + o, g + o, min(16384u, bytes - o), &bars[2]);
  };
  if (t == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 128);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  if (t == 0) {   // step n's weight images (hi, lo) and the first source tile
    const uint8_t* wsrc = a.wimg + (size_t)n * 2 * WB + moff;
    mbar_expect_tx(&bars[0], 2 * mbytes);
    for (uint32_t o = 0; o < mbytes; o += 16384u) {
      bulk_g2s(whi + o, wsrc + o, min(16384u, mbytes - o), &bars[0]);
      bulk_g2s(wlo + o, wsrc + WB + o, min(16384u, mbytes - o), &bars[0]);
    }
    if ((int)blockIdx.x < ntiles) prefetch(blockIdx.x);
  }
  const uint32_t idesc = idesc_bf16(128, Nc, false, NN);
  const int q = warp & 3, h = warp >> 2, rr = 32 * q + lane;
  const uint32_t lb = tm + ((uint32_t)(32 * q) << 16);
  const int cb = h * (Nc / 2), nch8 = Nc / 16;   // phase-1 columns: cb + 8j, j < nch8
  const float dt = a.dt;
  const float zc = -dt * driver_dfdz_coef(a.problem, a.lam), zc0 = -dt * driver_dfdz_const(a.problem);
  int j = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++j) {
    const int64_t i0 = (int64_t)tile * 128;
    // per-row operand scale (B1: ā_{n+1}); rows past B are zero (not copied)
    if (t < 128) {
      const int64_t m = i0 + t;
      srow[t] = m < a.B ? (OP == B1 ? abar_of(a, n, m) : 1.0f) : 0.0f;
    }
    mbar_wait(&bars[2], (uint32_t)(j & 1));
    __syncthreads();
    const int g4 = K / 4;
    for (int e = t; e < 128 * g4; e += RT) {
      const int r = e / g4, c = 4 * (e - r * g4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      const float sc = srow[r];
      if (sc != 0.0f) {
        v = *reinterpret_cast<const float4*>(rawt + r * K + c);
        v = make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w);
      }
      uint2 hi, lo;
      split4(v, hi, lo);
      *reinterpret_cast<uint2*>(ahi + ioff(r, c, K)) = hi;
      *reinterpret_cast<uint2*>(alo + ioff(r, c, K)) = lo;
    }
    fence_async_smem();
    tc_before();
    __syncthreads();   // images complete; the source tile is consumed
    if (t == 0) {
      tc_after();
      if (tile + (int)gridDim.x < ntiles) prefetch(tile + gridDim.x);
      if (j == 0) mbar_wait(&bars[0], 0);
      const Opnd Ah = kmaj(ahi, K), Al = kmaj(alo, K);
      const Opnd Wh = NN ? mnmaj(whi, Nc) : kmaj(whi, K), Wl = NN ? mnmaj(wlo, Nc) : kmaj(wlo, K);
      gemm(tm, Ah, Wh, K / 16, idesc, false);
      gemm(tm, Ah, Wl, K / 16, idesc, true);
      gemm(tm, Al, Wh, K / 16, idesc, true);
      mma_commit(&bars[1]);
    }
    mbar_wait(&bars[1], (uint32_t)(j & 1));
    tc_after();
    {   // phase 1: TMEM -> tile (lane = row), all loads in flight
      uint32_t r8[8][8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (jj < nch8) tmem_ld8_nowait(lb + (uint32_t)(cb + 8 * jj), r8[jj]);
      tmem_ld_wait();
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        if (jj >= nch8) break;
        reg_fence8(r8[jj]);
        float* dst = stile + rr * ldt + cb + 8 * jj;
        *reinterpret_cast<uint4*>(dst) = make_uint4(r8[jj][0], r8[jj][1], r8[jj][2], r8[jj][3]);
        *reinterpret_cast<uint4*>(dst + 4) = make_uint4(r8[jj][4], r8[jj][5], r8[jj][6], r8[jj][7]);
      }
    }
    tc_before();
    __syncthreads();   // the tile is complete; the accumulator may be overwritten
    // phase 2: warp w, rows w, w+8, ...; lane = columns 4·lane .. +3
    const int c4 = 4 * lane;
    const bool lane_on = c4 < Nc;
    for (int r = warp; r < 128; r += RT / 32) {
      const int64_t m = i0 + r;
      if (m >= a.B) break;
      const size_t row = (size_t)n * a.Bs + m;
      float4 v = lane_on ? *reinterpret_cast<const float4*>(stile + r * ldt + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (OP == F1 && lane_on)
        *reinterpret_cast<float4*>(a.H1 + row * Wp + c4) =
            make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
      if (OP == F2 && lane_on) {   // H2 = H1 + ReLU(A2)
        const float4 p = __ldg(reinterpret_cast<const float4*>(a.H1 + row * Wp + c4));
        *reinterpret_cast<float4*>(a.H2 + row * Wp + c4) =
            make_float4(p.x + fmaxf(v.x, 0.f), p.y + fmaxf(v.y, 0.f), p.z + fmaxf(v.z, 0.f),
                        p.w + fmaxf(v.w, 0.f));
      }
      if (OP == F3) {   // Z·ΔW, |Z|² | Σ Z; G = ΔW - Δt ∂_z f in place (R2)
        float s1 = 0.f, s2 = 0.f;
        if (lane_on) {
          float* gp = a.GW + row * Dp + c4;
          const float4 gv = *reinterpret_cast<const float4*>(gp);
          const float z[4] = {v.x, v.y, v.z, v.w};
          float g[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c4 + e >= d) { g[e] = 0.f; continue; }
            s1 = fmaf(z[e], g[e], s1);
            if (a.problem == kHJB) s2 = fmaf(z[e], z[e], s2);
            else if (a.problem == kBlackScholes) s2 += z[e];
            // ∂_z f = -λ z (HJB), r/σ (Black-Scholes), 0 (heat, Allen-Cahn)
            g[e] = fmaf(zc, z[e], g[e] + zc0);
          }
          if (!a.eval) *reinterpret_cast<float4*>(gp) = make_float4(g[0], g[1], g[2], g[3]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane == 0) *reinterpret_cast<float2*>(a.S + row * 2) = make_float2(s1, s2);
      }
      if (OP == B1 && lane_on) {   // dH2 -> DA; dA2 = dH2 ⊙ 1[A2 > 0] (A2 > 0 <=> H2 > H1, R15) -> DH
        const float4 h1 = __ldg(reinterpret_cast<const float4*>(a.H1 + row * Wp + c4));
        const float4 h2 = __ldg(reinterpret_cast<const float4*>(a.H2 + row * Wp + c4));
        *reinterpret_cast<float4*>(a.DA + row * Wp + c4) = v;
        *reinterpret_cast<float4*>(a.DH + row * Wp + c4) =
            make_float4(h2.x > h1.x ? v.x : 0.f, h2.y > h1.y ? v.y : 0.f, h2.z > h1.z ? v.z : 0.f,
                        h2.w > h1.w ? v.w : 0.f);
      }
      if (OP == B2 && lane_on) {   // dH1 = dH2 + dA2 W̃2; dA1 = dH1 ⊙ 1[H1 > 0] -> DA (over dH2)
        const float4 dh = *reinterpret_cast<const float4*>(a.DA + row * Wp + c4);
        const float4 h1 = __ldg(reinterpret_cast<const float4*>(a.H1 + row * Wp + c4));
        *reinterpret_cast<float4*>(a.DA + row * Wp + c4) =
            make_float4(h1.x > 0.f ? dh.x + v.x : 0.f, h1.y > 0.f ? dh.y + v.y : 0.f,
                        h1.z > 0.f ? dh.z + v.z : 0.f, h1.w > 0.f ? dh.w + v.w : 0.f);
      }
    }
    __syncthreads();   // the tile is read: the next tile's phase 1 may overwrite it
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 128);
  }
}

// The same row GEMMs with compile-time operand shapes (the built dims): one CTA per
// (128-row tile, step n), two CTAs per SM, so one CTA's loads overlap the other's MMAs
// and epilogue.  A is loaded from global with all of a thread's float4 loads in
// flight, converted to bf16 hi / lo in shared memory; the epilogue goes through a
// padded half tile that reuses the A images (free once the MMAs completed), then whole
// rows per warp (coalesced).
template <int OP, int DP, int WP>
__global__ void __launch_bounds__(RT, 2) k_rows_gemm_t(RowsArgs a) {
  constexpr int K = (OP == F1 || OP == B1) ? DP : WP, NC = (OP == F3) ? DP : WP;
  constexpr int G4 = K / 4, U = (128 * G4 + RT - 1) / RT, LDT = NC + 4, NCH8 = NC / 16;
  constexpr uint32_t MB = (uint32_t)NC * K * 2, AB = 128u * K * 2;
  // the half tile reuses the A images when it fits them (the built large shapes), else
  // it has its own region after them (small shapes)
  constexpr bool ALIAS = 64 * LDT * 4 <= 2 * AB;
  constexpr int mat = (OP == F1) ? 0 : (OP == F2 || OP == B2) ? 1 : 2;
  constexpr bool NN = OP == B1 || OP == B2;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[3];   // 0 weights, 1 MMA, 2 A image (F3)
  // F3 reads H2 as the tile image F12 wrote (no conversion)
  constexpr bool IMGA = OP == F3;
  __shared__ uint32_t tslot;
  __shared__ float srow[128];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int n = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * 128;
  const int d = a.d;
  const float* src = OP == F1 ? a.XT : OP == F2 ? a.H1 : OP == F3 ? a.H2 : OP == B1 ? a.GW : a.DH;
  constexpr uint32_t WB = 2u * (WP * DP + WP * WP + DP * WP);
  constexpr uint32_t moff = mat == 0 ? 0u : mat == 1 ? 2u * WP * DP : 2u * (WP * DP + WP * WP);
  uint8_t* whi = sm;
  uint8_t* wlo = sm + MB;
  uint8_t* ahi = sm + 2 * MB;
  uint8_t* alo = ahi + AB;
  float* stile = reinterpret_cast<float*>(ALIAS ? ahi : alo + AB);
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 128);
  if (t < 128) {
    const int64_t m = i0 + t;
    srow[t] = m < a.B ? (OP == B1 ? abar_of(a, n, m) : 1.0f) : 0.0f;
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  if (t == 0) {
    const uint8_t* wsrc = a.wimg + (size_t)n * 2 * WB + moff;
    mbar_expect_tx(&bars[0], 2 * MB);
    for (uint32_t o = 0; o < MB; o += 16384u) {
      bulk_g2s(whi + o, wsrc + o, min(16384u, MB - o), &bars[0]);
      bulk_g2s(wlo + o, wsrc + WB + o, min(16384u, MB - o), &bars[0]);
    }
    if (IMGA) {   // the tile's hi / lo image straight into the A operand
      constexpr uint32_t IB = 128u * K * 2;
      const uint8_t* g = tile_img(src, a, n, i0, K);
      mbar_expect_tx(&bars[2], 2 * IB);
      for (uint32_t o = 0; o < IB; o += 16384u) {
        bulk_g2s(ahi + o, g + o, min(16384u, IB - o), &bars[2]);
        bulk_g2s(alo + o, g + IB + o, min(16384u, IB - o), &bars[2]);
      }
    }
  }
  // F3: this warp's G rows of half tile 0 (rows warp + 8j) in flight during the bulk
  // copies and the MMAs; half 1's are issued once half 0's rows are done
  constexpr int NRH = 64 / (RT / 32);   // rows per warp and half tile
  const int c4 = 4 * lane;
  const bool lane_on = c4 < NC;
  float4 gq0[OP == F3 ? NRH : 1];
  auto load_g = [&](int hf, float4 (&gq)[OP == F3 ? NRH : 1]) {
#pragma unroll
    for (int j = 0; j < (OP == F3 ? NRH : 0); ++j) {
      const int64_t m = i0 + 64 * hf + warp + 8 * j;
      gq[j] = (m < a.B && lane_on)
                  ? __ldcs(reinterpret_cast<const float4*>(a.GW + ((size_t)n * a.Bs + (size_t)m) * DP + c4))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if constexpr (OP == F3) load_g(0, gq0);
  // stage A: all U float4 loads in flight, then split / store
  if constexpr (!IMGA) {
    const float* base = src + ((size_t)n * a.Bs + i0) * K;
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = t + u * RT;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      int r, c;
      slot_rc<K>(e, r, c);
      if (e < 128 * G4 && srow[r] != 0.0f) v[u] = __ldg(reinterpret_cast<const float4*>(base + r * K + c));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = t + u * RT;
      if (e >= 128 * G4) break;
      int r, c;
      slot_rc<K>(e, r, c);
      const float sc = srow[r];
      uint2 hi, lo;
      split4(make_float4(sc * v[u].x, sc * v[u].y, sc * v[u].z, sc * v[u].w), hi, lo);
      *reinterpret_cast<uint2*>(ahi + ioff(r, c, K)) = hi;
      *reinterpret_cast<uint2*>(alo + ioff(r, c, K)) = lo;
    }
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (t == 0) {
    tc_after();
    mbar_wait(&bars[0], 0);
    if (IMGA) mbar_wait(&bars[2], 0);
    constexpr uint32_t idesc = idesc_bf16(128, NC, false, NN);
    const Opnd Ah = kmaj(ahi, K), Al = kmaj(alo, K);
    const Opnd Wh = NN ? mnmaj(whi, NC) : kmaj(whi, K), Wl = NN ? mnmaj(wlo, NC) : kmaj(wlo, K);
    gemm(tm, Ah, Wh, K / 16, idesc, false);
    gemm(tm, Ah, Wl, K / 16, idesc, true);
    gemm(tm, Al, Wh, K / 16, idesc, true);
    mma_commit(&bars[1]);
  }
  mbar_wait(&bars[1], 0);
  tc_after();
  const int q = warp & 3, h = warp >> 2;
  const uint32_t lb = tm + ((uint32_t)(32 * q) << 16);
  const int cb = h * (NC / 2);
  const float dt = a.dt;
  const float zc = -dt * driver_dfdz_coef(a.problem, a.lam), zc0 = -dt * driver_dfdz_const(a.problem);
  if constexpr (OP == F3) {
    // the epilogue from the prefetched G rows: no memory round trip per row batch
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      if ((q >> 1) == hf) {   // phase 1: this half's lane quadrants -> tile rows 0..63
        uint32_t r8[NCH8][8];
#pragma unroll
        for (int jj = 0; jj < NCH8; ++jj) tmem_ld8_nowait(lb + (uint32_t)(cb + 8 * jj), r8[jj]);
        tmem_ld_wait();
        const int rl = 32 * (q & 1) + lane;
#pragma unroll
        for (int jj = 0; jj < NCH8; ++jj) {
          reg_fence8(r8[jj]);
          float* dstp = stile + rl * LDT + cb + 8 * jj;
          *reinterpret_cast<uint4*>(dstp) = make_uint4(r8[jj][0], r8[jj][1], r8[jj][2], r8[jj][3]);
          *reinterpret_cast<uint4*>(dstp + 4) = make_uint4(r8[jj][4], r8[jj][5], r8[jj][6], r8[jj][7]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NRH; ++j) {
        const int r = warp + 8 * j;
        const int64_t m = i0 + 64 * hf + r;
        if (m >= a.B) continue;   // warp-uniform
        const size_t row = (size_t)n * a.Bs + (size_t)m;
        const float4 v = lane_on ? *reinterpret_cast<const float4*>(stile + r * LDT + c4)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        float s1 = 0.f, s2 = 0.f;
        if (lane_on) {   // Z·ΔW, |Z|² | Σ Z; G = ΔW - Δt ∂_z f in place (R2)
          const float4 gv = gq0[j];
          const float z[4] = {v.x, v.y, v.z, v.w};
          float g[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c4 + e >= d) { g[e] = 0.f; continue; }
            s1 = fmaf(z[e], g[e], s1);
            if (a.problem == kHJB) s2 = fmaf(z[e], z[e], s2);
            else if (a.problem == kBlackScholes) s2 += z[e];
            g[e] = fmaf(zc, z[e], g[e] + zc0);   // ∂_z f = -λ z (HJB), r/σ (Black-Scholes)
          }
          if (!a.eval) *reinterpret_cast<float4*>(a.GW + row * DP + c4) = make_float4(g[0], g[1], g[2], g[3]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane == 0) *reinterpret_cast<float2*>(a.S + row * 2) = make_float2(s1, s2);
      }
      if (hf == 0) load_g(1, gq0);   // half 1's rows, in flight over its phase 1
      __syncthreads();
    }
  } else {
#pragma unroll 1
  for (int hf = 0; hf < 2; ++hf) {
    if ((q >> 1) == hf) {   // phase 1: this half's lane quadrants -> tile rows 0..63
      uint32_t r8[NCH8][8];
#pragma unroll
      for (int jj = 0; jj < NCH8; ++jj) tmem_ld8_nowait(lb + (uint32_t)(cb + 8 * jj), r8[jj]);
      tmem_ld_wait();
      const int rl = 32 * (q & 1) + lane;
#pragma unroll
      for (int jj = 0; jj < NCH8; ++jj) {
        reg_fence8(r8[jj]);
        float* dstp = stile + rl * LDT + cb + 8 * jj;
        *reinterpret_cast<uint4*>(dstp) = make_uint4(r8[jj][0], r8[jj][1], r8[jj][2], r8[jj][3]);
        *reinterpret_cast<uint4*>(dstp + 4) = make_uint4(r8[jj][4], r8[jj][5], r8[jj][6], r8[jj][7]);
      }
    }
    __syncthreads();
    // phase 2: warp w, half-tile rows w, w+8, ...; lane = columns 4·lane .. +3.  Rows
    // go in batches of RB whose global inputs (H1, H2, G, dH2) are loaded together, so
    // a warp waits one memory round trip per batch, not per row
    constexpr int RB = 4;
#pragma unroll 1
    for (int r0 = warp; r0 < 64; r0 += RB * (RT / 32)) {
      float4 pa[RB], pb[RB];
      size_t rws[RB];
      bool ok[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = r0 + k * (RT / 32);
        const int64_t m = i0 + 64 * hf + r;
        ok[k] = r < 64 && m < a.B;
        rws[k] = (size_t)n * a.Bs + (size_t)(ok[k] ? m : 0);
        pa[k] = pb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok[k] && lane_on) {
          if (OP == F2 || OP == B1 || OP == B2) pa[k] = __ldg(reinterpret_cast<const float4*>(a.H1 + rws[k] * WP + c4));
          if (OP == F3) pa[k] = *reinterpret_cast<const float4*>(a.GW + rws[k] * DP + c4);
          if (OP == B1) pb[k] = __ldg(reinterpret_cast<const float4*>(a.H2 + rws[k] * WP + c4));
          if (OP == B2) pb[k] = *reinterpret_cast<const float4*>(a.DA + rws[k] * WP + c4);
        }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
      if (!ok[k]) continue;   // warp-uniform
      const int r = r0 + k * (RT / 32);
      const size_t row = rws[k];
      const float4 v = lane_on ? *reinterpret_cast<const float4*>(stile + r * LDT + c4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
      if (OP == F1 || OP == F2) {   // ReLU masks 1[A > 0] of the row for the fused adjoint
        const uint32_t b0 = __ballot_sync(0xffffffffu, lane_on && v.x > 0.f);
        const uint32_t b1 = __ballot_sync(0xffffffffu, lane_on && v.y > 0.f);
        const uint32_t b2 = __ballot_sync(0xffffffffu, lane_on && v.z > 0.f);
        const uint32_t b3 = __ballot_sync(0xffffffffu, lane_on && v.w > 0.f);
        if (lane == 0 && !a.eval)
          *reinterpret_cast<uint4*>((OP == F1 ? a.M1 : a.M2) + row * 4) = make_uint4(b0, b1, b2, b3);
      }
      if (OP == F1 && lane_on)
        *reinterpret_cast<float4*>(a.H1 + row * WP + c4) =
            make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
      if (OP == F2 && lane_on) {   // H2 = H1 + ReLU(A2)
        const float4 p = pa[k];
        *reinterpret_cast<float4*>(a.H2 + row * WP + c4) =
            make_float4(p.x + fmaxf(v.x, 0.f), p.y + fmaxf(v.y, 0.f), p.z + fmaxf(v.z, 0.f),
                        p.w + fmaxf(v.w, 0.f));
      }
      if (OP == F3) {   // Z·ΔW, |Z|² | Σ Z; G = ΔW - Δt ∂_z f in place (R2)
        float s1 = 0.f, s2 = 0.f;
        if (lane_on) {
          float* gp = a.GW + row * DP + c4;
          const float4 gv = pa[k];
          const float z[4] = {v.x, v.y, v.z, v.w};
          float g[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c4 + e >= d) { g[e] = 0.f; continue; }
            s1 = fmaf(z[e], g[e], s1);
            if (a.problem == kHJB) s2 = fmaf(z[e], z[e], s2);
            else if (a.problem == kBlackScholes) s2 += z[e];
            g[e] = fmaf(zc, z[e], g[e] + zc0);   // ∂_z f = -λ z (HJB), r/σ (Black-Scholes)
          }
          if (!a.eval) *reinterpret_cast<float4*>(gp) = make_float4(g[0], g[1], g[2], g[3]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane == 0) *reinterpret_cast<float2*>(a.S + row * 2) = make_float2(s1, s2);
      }
      if (OP == B1 && lane_on) {   // dH2 -> DA; dA2 = dH2 ⊙ 1[A2 > 0] (H2 > H1, R15) -> DH
        const float4 h1 = pa[k], h2 = pb[k];
        *reinterpret_cast<float4*>(a.DA + row * WP + c4) = v;
        *reinterpret_cast<float4*>(a.DH + row * WP + c4) =
            make_float4(h2.x > h1.x ? v.x : 0.f, h2.y > h1.y ? v.y : 0.f, h2.z > h1.z ? v.z : 0.f,
                        h2.w > h1.w ? v.w : 0.f);
      }
      if (OP == B2 && lane_on) {   // dH1 = dH2 + dA2 W̃2; dA1 = dH1 ⊙ 1[H1 > 0] -> DA
        const float4 dh = pb[k], h1 = pa[k];
        *reinterpret_cast<float4*>(a.DA + row * WP + c4) =
            make_float4(h1.x > 0.f ? dh.x + v.x : 0.f, h1.y > 0.f ? dh.y + v.y : 0.f,
                        h1.z > 0.f ? dh.z + v.z : 0.f, h1.w > 0.f ? dh.w + v.w : 0.f);
      }
    }
      }
    __syncthreads();
  }
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 128);
  }
}

// ------------------------------------------------------------------ fused forward F1 + F2
// Compile-time shapes: one CTA per SM walks a contiguous range of the (step n, 128-row
// tile) items in step-major order (one wave at any N; a grid of ⌊#SM/N⌋ × N CTAs left
// 68 SMs idle at N = 80) with the step's W̃1 and W̃2 (hi / lo) resident, reloaded when
// the range crosses a step, the next item's X̃ rows in flight:
//   G1  A1 = X̃ W̃1ᵀ   (X̃ converted from the fp32 rows the path kernel wrote; its image
//                     replaces them in place, for dW̃1)
//   E1  H1 = ReLU(A1): the G2 operand (shared memory) and the H1 image (for dW̃2), mask
//       1[A1 > 0]; H1 stays in the registers of its TMEM lane for E2
//   G2  A2 = H1 W̃2ᵀ
//   E2  H2 = H1 + ReLU(A2): the H2 image (F3's A operand, dW̃3), mask 1[A2 > 0]
// Thread (lane quadrant q, column half h) owns row 32q + lane and writes its half row of
// each image as 16-byte chunks straight to memory (8 consecutive rows per 128 bytes).
template <int DP, int WP>
__global__ void __launch_bounds__(RT, 1) k_rows_f12_t(RowsArgs a) {
  constexpr int G4N = DP / 4, U = (128 * G4N + RT - 1) / RT, NCH8 = WP / 16;
  constexpr int KM = DP > WP ? DP : WP;
  constexpr uint32_t MB1 = (uint32_t)WP * DP * 2, MB2 = (uint32_t)WP * WP * 2, AB = 128u * KM * 2;
  constexpr uint32_t WB = 2u * (WP * DP + WP * WP + DP * WP);
  constexpr uint32_t XIMG = 128u * DP * 2, HIMG = 128u * WP * 2;   // bytes of one hi (or lo) image
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[2];   // 0 weights, 1 MMA
  __shared__ uint32_t tslot;
  __shared__ __align__(16) uint32_t mk[2][128][4];   // mask words per column half (disjoint bits)
  uint8_t* w1h = sm;
  uint8_t* w1l = sm + MB1;
  uint8_t* w2h = sm + 2 * MB1;
  uint8_t* w2l = w2h + MB2;
  uint8_t* ahi = w2l + MB2;
  uint8_t* alo = ahi + AB;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // (step, tile) items in step-major order, a contiguous range per CTA (one wave of one
  // CTA per SM at any N; the weights are reloaded when the range crosses a step)
  const int ntiles = (int)((a.B + 127) / 128);
  const int64_t items = (int64_t)a.N * ntiles;
  const int64_t it0 = blockIdx.x * items / gridDim.x, it1 = (blockIdx.x + 1) * items / gridDim.x;
  int n = (int)(it0 / ntiles);
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
  auto load_w = [&](int nn) {   // step nn's W̃1 and W̃2 (hi, lo); thread 0
    const uint8_t* wsrc = a.wimg + (size_t)nn * 2 * WB;
    const uint32_t o2 = MB1;
    mbar_expect_tx(&bars[0], 2 * (MB1 + MB2));
    for (uint32_t o = 0; o < MB1; o += 16384u) {
      bulk_g2s(w1h + o, wsrc + o, min(16384u, MB1 - o), &bars[0]);
      bulk_g2s(w1l + o, wsrc + WB + o, min(16384u, MB1 - o), &bars[0]);
    }
    for (uint32_t o = 0; o < MB2; o += 16384u) {
      bulk_g2s(w2h + o, wsrc + o2 + o, min(16384u, MB2 - o), &bars[0]);
      bulk_g2s(w2l + o, wsrc + WB + o2 + o, min(16384u, MB2 - o), &bars[0]);
    }
  };
  if (t == 0 && it0 < it1) load_w(n);
  const int q = warp & 3, h = warp >> 2, rr = 32 * q + lane;
  const uint32_t lb = tm + ((uint32_t)(32 * q) << 16);
  const int cb = h * (WP / 2);
  constexpr uint32_t idesc = idesc_bf16(128, WP, false, false);
  const bool store = !a.eval;
  float4 v[U];
  auto load = [&](int nn, int tile) {   // X̃ rows of item (nn, tile) (fp32, from the path kernel)
    const int64_t i0 = (int64_t)tile * 128;
    const float* base = a.XT + ((size_t)nn * a.Bs + i0) * DP;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = t + u * RT;
      int r, c;
      slot_rc<DP>(e, r, c);
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < 128 * G4N && i0 + r < a.B) v[u] = __ldg(reinterpret_cast<const float4*>(base + r * DP + c));
    }
  };
  auto out_masks = [&](int64_t i0, uint32_t* mdst) {   // 4 words per row, one row per lane
    if (!store || lane >= 16) return;
    const int r = 16 * warp + lane;
    if (i0 + r >= a.B) return;
    const uint4 m0 = *reinterpret_cast<const uint4*>(mk[0][r]), m1 = *reinterpret_cast<const uint4*>(mk[1][r]);
    *reinterpret_cast<uint4*>(mdst + ((size_t)n * a.Bs + i0 + r) * 4) =
        make_uint4(m0.x | m1.x, m0.y | m1.y, m0.z | m1.z, m0.w | m1.w);
  };
  float h1[NCH8 * 8];   // H1 of this thread's row and column half (E1 -> E2)
  uint32_t mph = 0, wph = 0;
  bool wait_w = true;   // the weights of step n are being loaded
  int tile = (int)(it0 - (int64_t)n * ntiles);
  if (it0 < it1) load(n, tile);
  for (int64_t item = it0; item < it1; ++item) {
    const int nn = tile + 1 == ntiles ? n + 1 : n, ntile = tile + 1 == ntiles ? 0 : tile + 1;
    const int64_t i0 = (int64_t)tile * 128;
    // X̃ -> bf16 hi / lo A image (K = DP), and the same bytes over the tile's fp32 rows
    // in memory (the X̃ image of dW̃1; a warp writes two whole 128-byte core matrices)
    uint8_t* xd = tile_img(a.XT, a, n, i0, DP);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = t + u * RT;
      if (e >= 128 * G4N) break;
      int r, c;
      slot_rc<DP>(e, r, c);
      uint2 hi, lo;
      split4(v[u], hi, lo);
      const uint32_t o = ioff(r, c, DP);
      *reinterpret_cast<uint2*>(ahi + o) = hi;
      *reinterpret_cast<uint2*>(alo + o) = lo;
      if (store) {
        *reinterpret_cast<uint2*>(xd + o) = hi;
        *reinterpret_cast<uint2*>(xd + XIMG + o) = lo;
      }
    }
    if (item + 1 < it1) load(nn, ntile);   // in flight until the next item
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (t == 0) {   // G1: A1 = X̃ W̃1ᵀ; the X̃ image over this tile's fp32 rows (for dW̃1)
      tc_after();
      if (wait_w) { mbar_wait(&bars[0], wph); wph ^= 1; }
      const Opnd Ah = kmaj(ahi, DP), Al = kmaj(alo, DP), Wh = kmaj(w1h, DP), Wl = kmaj(w1l, DP);
      gemm(tm, Ah, Wh, DP / 16, idesc, false);
      gemm(tm, Ah, Wl, DP / 16, idesc, true);
      gemm(tm, Al, Wh, DP / 16, idesc, true);
      mma_commit(&bars[1]);
    }
    wait_w = false;
    mbar_wait(&bars[1], mph);
    mph ^= 1;
    tc_after();
    // ---- E1 (every thread: its half row)
    {
      uint8_t* hd = tile_img(a.H1, a, n, i0, WP);
      uint32_t r8[NCH8][8];
#pragma unroll
      for (int jj = 0; jj < NCH8; ++jj) tmem_ld8_nowait(lb + (uint32_t)(cb + 8 * jj), r8[jj]);
      tmem_ld_wait();
      uint32_t bits[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int jj = 0; jj < NCH8; ++jj) {
        reg_fence8(r8[jj]);
        const int c0 = cb + 8 * jj;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float x = __uint_as_float(r8[jj][j]);
          h1[8 * jj + j] = fmaxf(x, 0.0f);
          bits[j & 3] |= (x > 0.0f ? 1u : 0u) << ((c0 + j) >> 2);
        }
        const float* f = h1 + 8 * jj;
        uint2 h0, l0, hh1, l1;
        split4(make_float4(f[0], f[1], f[2], f[3]), h0, l0);
        split4(make_float4(f[4], f[5], f[6], f[7]), hh1, l1);
        const uint32_t o = ioff(rr, c0, WP);
        const uint4 hv = make_uint4(h0.x, h0.y, hh1.x, hh1.y), lv = make_uint4(l0.x, l0.y, l1.x, l1.y);
        *reinterpret_cast<uint4*>(ahi + o) = hv;
        *reinterpret_cast<uint4*>(alo + o) = lv;
        if (store) {
          *reinterpret_cast<uint4*>(hd + o) = hv;
          *reinterpret_cast<uint4*>(hd + HIMG + o) = lv;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) mk[h][rr][e] = bits[e];
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (t == 0) {   // G2: A2 = H1 W̃2ᵀ
      tc_after();
      const Opnd Ah = kmaj(ahi, WP), Al = kmaj(alo, WP), Wh = kmaj(w2h, WP), Wl = kmaj(w2l, WP);
      gemm(tm, Ah, Wh, WP / 16, idesc, false);
      gemm(tm, Ah, Wl, WP / 16, idesc, true);
      gemm(tm, Al, Wh, WP / 16, idesc, true);
      mma_commit(&bars[1]);
    }
    out_masks(i0, a.M1);
    mbar_wait(&bars[1], mph);
    mph ^= 1;
    tc_after();
    __syncthreads();   // mask words read before E2 rewrites them
    // ---- E2
    {
      uint8_t* hd = tile_img(a.H2, a, n, i0, WP);
      uint32_t r8[NCH8][8];
#pragma unroll
      for (int jj = 0; jj < NCH8; ++jj) tmem_ld8_nowait(lb + (uint32_t)(cb + 8 * jj), r8[jj]);
      tmem_ld_wait();
      uint32_t bits[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int jj = 0; jj < NCH8; ++jj) {
        reg_fence8(r8[jj]);
        const int c0 = cb + 8 * jj;
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float x = __uint_as_float(r8[jj][j]);
          f[j] = h1[8 * jj + j] + fmaxf(x, 0.0f);
          bits[j & 3] |= (x > 0.0f ? 1u : 0u) << ((c0 + j) >> 2);
        }
        uint2 h0, l0, hh1, l1;
        split4(make_float4(f[0], f[1], f[2], f[3]), h0, l0);
        split4(make_float4(f[4], f[5], f[6], f[7]), hh1, l1);
        const uint32_t o = ioff(rr, c0, WP);
        *reinterpret_cast<uint4*>(hd + o) = make_uint4(h0.x, h0.y, hh1.x, hh1.y);
        *reinterpret_cast<uint4*>(hd + HIMG + o) = make_uint4(l0.x, l0.y, l1.x, l1.y);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) mk[h][rr][e] = bits[e];
    }
    tc_before();
    __syncthreads();
    out_masks(i0, a.M2);
    __syncthreads();   // mask words read before the next tile's E1
    if (item + 1 < it1 && nn != n) {   // G1 and G2 of step n have completed: its weights are free
      if (t == 0) load_w(nn);
      wait_w = true;
    }
    n = nn;
    tile = ntile;
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 128);
  }
}

// ------------------------------------------------------------------ fused adjoint B1 + B2
// Compile-time shapes: one CTA per SM walks a contiguous range of the (step n, 128-row
// tile) items in step-major order with the step's W̃3 and W̃2 images (hi / lo) resident
// (reloaded when the range crosses a step), the next item's G rows in flight while the
// current one computes:
//   G4  dH2 = dZ W̃3, dZ = ā_{n+1} G (staged as bf16 hi / lo; its image replaces the
//       tile's G rows in place, the A operand of dW̃3)
//   E4  dA2 = dH2 ⊙ 1[A2 > 0] (mask words from F2): the dA2 image (dW̃2) and, in shared
//       memory, the A operand of G6 (over the dZ images, which G4 has read)
//   G6  dH1 = dH2 + dA2 W̃2 (accumulated onto dH2 in TMEM)
//   E6  dA1 = dH1 ⊙ 1[A1 > 0] (mask words from F1): the dA1 image (dW̃1)
// dH2 never leaves the chip; every thread writes its half row of the images directly.
template <int DP, int WP>
__global__ void __launch_bounds__(RT, 1) k_rows_b12_t(RowsArgs a) {
  constexpr int G4N = DP / 4, U = (128 * G4N + RT - 1) / RT, NCH8 = WP / 16;
  constexpr int KM = DP > WP ? DP : WP;
  constexpr uint32_t MB3 = (uint32_t)DP * WP * 2, MB2 = (uint32_t)WP * WP * 2, AB = 128u * KM * 2;
  constexpr uint32_t WB = 2u * (WP * DP + WP * WP + DP * WP);
  constexpr uint32_t ZIMG = 128u * DP * 2, HIMG = 128u * WP * 2;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[2];   // 0 weights, 1 MMA
  __shared__ uint32_t tslot;
  __shared__ float srow[128];
  uint8_t* w3h = sm;
  uint8_t* w3l = sm + MB3;
  uint8_t* w2h = sm + 2 * MB3;
  uint8_t* w2l = w2h + MB2;
  uint8_t* ahi = w2l + MB2;
  uint8_t* alo = ahi + AB;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // (step, tile) items in step-major order, a contiguous range per CTA (one wave of one
  // CTA per SM at any N; the weights are reloaded when the range crosses a step)
  const int ntiles = (int)((a.B + 127) / 128);
  const int64_t items = (int64_t)a.N * ntiles;
  const int64_t it0 = blockIdx.x * items / gridDim.x, it1 = (blockIdx.x + 1) * items / gridDim.x;
  int n = (int)(it0 / ntiles);
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
  auto load_w = [&](int nn) {   // step nn's W̃3 and W̃2 (hi, lo); thread 0
    const uint8_t* wsrc = a.wimg + (size_t)nn * 2 * WB;
    const uint32_t o3 = 2u * (WP * DP + WP * WP), o2 = 2u * WP * DP;
    mbar_expect_tx(&bars[0], 2 * (MB3 + MB2));
    for (uint32_t o = 0; o < MB3; o += 16384u) {
      bulk_g2s(w3h + o, wsrc + o3 + o, min(16384u, MB3 - o), &bars[0]);
      bulk_g2s(w3l + o, wsrc + WB + o3 + o, min(16384u, MB3 - o), &bars[0]);
    }
    for (uint32_t o = 0; o < MB2; o += 16384u) {
      bulk_g2s(w2h + o, wsrc + o2 + o, min(16384u, MB2 - o), &bars[0]);
      bulk_g2s(w2l + o, wsrc + WB + o2 + o, min(16384u, MB2 - o), &bars[0]);
    }
  };
  if (t == 0 && it0 < it1) load_w(n);
  const int q = warp & 3, h = warp >> 2, rr = 32 * q + lane;
  const uint32_t lb = tm + ((uint32_t)(32 * q) << 16);
  const int cb = h * (WP / 2);
  constexpr uint32_t idesc = idesc_bf16(128, WP, false, true);
  float4 v[U];
  auto load = [&](int nn, int tile) {   // G rows of item (nn, tile), all loads in flight
    const int64_t i0 = (int64_t)tile * 128;
    const float* base = a.GW + ((size_t)nn * a.Bs + i0) * DP;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = t + u * RT;
      int r, c;
      slot_rc<DP>(e, r, c);
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < 128 * G4N && i0 + r < a.B) v[u] = __ldg(reinterpret_cast<const float4*>(base + r * DP + c));
    }
  };
  // E4 / E6 on the accumulator: mask, then the half row's bf16 hi / lo chunks -> the
  // image at dst (and, for E4, the G6 operand in shared memory)
  auto epilogue = [&](const uint4& mk, uint8_t* dst, bool smem_img) {
    const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
    uint32_t r8[NCH8][8];
#pragma unroll
    for (int jj = 0; jj < NCH8; ++jj) tmem_ld8_nowait(lb + (uint32_t)(cb + 8 * jj), r8[jj]);
    tmem_ld_wait();
#pragma unroll
    for (int jj = 0; jj < NCH8; ++jj) {
      reg_fence8(r8[jj]);
      const int c0 = cb + 8 * jj;
      float f[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = c0 + j;
        f[j] = ((mw[col & 3] >> (col >> 2)) & 1u) ? __uint_as_float(r8[jj][j]) : 0.0f;
      }
      uint2 h0, l0, h1, l1;
      split4(make_float4(f[0], f[1], f[2], f[3]), h0, l0);
      split4(make_float4(f[4], f[5], f[6], f[7]), h1, l1);
      const uint32_t o = ioff(rr, c0, WP);
      const uint4 hv = make_uint4(h0.x, h0.y, h1.x, h1.y), lv = make_uint4(l0.x, l0.y, l1.x, l1.y);
      if (smem_img) {
        *reinterpret_cast<uint4*>(ahi + o) = hv;
        *reinterpret_cast<uint4*>(alo + o) = lv;
      }
      *reinterpret_cast<uint4*>(dst + o) = hv;
      *reinterpret_cast<uint4*>(dst + HIMG + o) = lv;
    }
  };
  // ā_{n+1} of a tile's rows (threads t < 128), loaded one tile ahead like G
  float pab = 0.0f, ppn = 1.0f;
  auto load_ab = [&](int nn, int tile) {
    const int64_t m = (int64_t)tile * 128 + t;
    if (t < 128 && m < a.B) {
      pab = __ldg(a.abar + m);
      ppn = per_step_abar(a.problem) ? __ldg(a.Pstore + (int64_t)nn * a.B + m) : 1.0f;
    } else {
      pab = 0.0f;
      ppn = 1.0f;
    }
  };
  // this thread's row masks (TMEM lane layout: row rr), also one tile ahead
  uint4 mk1n = make_uint4(0, 0, 0, 0), mk2n = make_uint4(0, 0, 0, 0);
  auto load_mk = [&](int nn, int tile) {
    const int64_t mrow = (int64_t)tile * 128 + rr;
    const size_t ro = ((size_t)nn * a.Bs + (size_t)mrow) * 4;
    const bool ok = mrow < a.B;
    mk2n = ok ? __ldg(reinterpret_cast<const uint4*>(a.M2 + ro)) : make_uint4(0, 0, 0, 0);
    mk1n = ok ? __ldg(reinterpret_cast<const uint4*>(a.M1 + ro)) : make_uint4(0, 0, 0, 0);
  };
  uint32_t mph = 0, wph = 0;
  bool wait_w = true;   // the weights of step n are being loaded
  int tile = (int)(it0 - (int64_t)n * ntiles);
  if (it0 < it1) { load(n, tile); load_ab(n, tile); load_mk(n, tile); }
  for (int64_t item = it0; item < it1; ++item) {
    const int nn = tile + 1 == ntiles ? n + 1 : n, ntile = tile + 1 == ntiles ? 0 : tile + 1;
    const int64_t i0 = (int64_t)tile * 128;
    if (t < 128) srow[t] = __fdividef(pab, ppn);   // 0 past B (pab = 0)
    __syncthreads();
    // dZ = ā_{n+1} G -> bf16 hi / lo A image (K = DP), and the same bytes over the
    // tile's G rows in memory (the dZ image of dW̃3)
    uint8_t* zd = tile_img(a.GW, a, n, i0, DP);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = t + u * RT;
      if (e >= 128 * G4N) break;
      int r, c;
      slot_rc<DP>(e, r, c);
      const float sc = srow[r];
      uint2 hi, lo;
      split4(make_float4(sc * v[u].x, sc * v[u].y, sc * v[u].z, sc * v[u].w), hi, lo);
      const uint32_t o = ioff(r, c, DP);
      *reinterpret_cast<uint2*>(ahi + o) = hi;
      *reinterpret_cast<uint2*>(alo + o) = lo;
      *reinterpret_cast<uint2*>(zd + o) = hi;
      *reinterpret_cast<uint2*>(zd + ZIMG + o) = lo;
    }
    const uint4 mk1 = mk1n, mk2 = mk2n;
    if (item + 1 < it1) {   // in flight until the next item
      load(nn, ntile);
      load_ab(nn, ntile);
      load_mk(nn, ntile);
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (t == 0) {   // G4: dH2 = dZ W̃3; the dZ image over this tile's G rows (for dW̃3)
      tc_after();
      if (wait_w) { mbar_wait(&bars[0], wph); wph ^= 1; }
      const Opnd Ah = kmaj(ahi, DP), Al = kmaj(alo, DP), Wh = mnmaj(w3h, WP), Wl = mnmaj(w3l, WP);
      gemm(tm, Ah, Wh, DP / 16, idesc, false);
      gemm(tm, Ah, Wl, DP / 16, idesc, true);
      gemm(tm, Al, Wh, DP / 16, idesc, true);
      mma_commit(&bars[1]);
    }
    wait_w = false;
    mbar_wait(&bars[1], mph);
    mph ^= 1;
    tc_after();
    epilogue(mk2, tile_img(a.DH, a, n, i0, WP), true);   // E4: dA2
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (t == 0) {   // G6: dH1 = dH2 + dA2 W̃2
      tc_after();
      const Opnd Ah = kmaj(ahi, WP), Al = kmaj(alo, WP), Wh = mnmaj(w2h, WP), Wl = mnmaj(w2l, WP);
      gemm(tm, Ah, Wh, WP / 16, idesc, true);
      gemm(tm, Ah, Wl, WP / 16, idesc, true);
      gemm(tm, Al, Wh, WP / 16, idesc, true);
      mma_commit(&bars[1]);
    }
    mbar_wait(&bars[1], mph);
    mph ^= 1;
    tc_after();
    epilogue(mk1, tile_img(a.DA, a, n, i0, WP), false);   // E6: dA1
    tc_before();
    __syncthreads();   // accumulator and A images read before the next tile
    if (item + 1 < it1 && nn != n) {   // G4 and G6 of step n have completed: its weights are free
      if (t == 0) load_w(nn);
      wait_w = true;
    }
    n = nn;
    tile = ntile;
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
      const float2 s = *reinterpret_cast<const float2*>(a.S + ((size_t)n * a.Bs + m) * 2);
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
// [r0, r1) of step n = blockIdx.z; M = 128 (output rows p < P), N = Q, K = TK rows a
// chunk.  Both fp32 sources are contiguous per chunk ([N][B][cols] buffers): bulk copies
// two chunks ahead, converted to MN-major bf16 hi / lo images, three MMA passes.
constexpr int TK = 64;
__global__ void __launch_bounds__(RT, 1) k_rows_tn(RowsArgs a, int rows_per_cta) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[3];   // MMA, raw[0], raw[1]
  __shared__ uint32_t tslot;
  __shared__ float srow[TK];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int which = blockIdx.y, n = blockIdx.z;
  const int Dp = a.Dp, Wp = a.Wp, d = a.d, w = a.w;
  const int P = which == 2 ? Dp : Wp, Q = which == 0 ? Dp : Wp;   // source row strides
  const float* srcA = which == 0 ? a.DA : which == 1 ? a.DH : a.GW;
  const float* srcB = which == 0 ? a.XT : which == 1 ? a.H1 : a.H2;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = (a.B < r0 + rows_per_cta ? a.B : r0 + rows_per_cta);
  const uint32_t AB = img_bytes(TK, 128), BB = img_bytes(TK, Q);
  uint8_t* aimg = sm;                          // A hi, A lo [TK × 128]
  uint8_t* bimg = sm + 2 * AB;                 // B hi, B lo [TK × Q]
  float* rawA0 = reinterpret_cast<float*>(bimg + 2 * img_bytes(TK, 128));
  float* rawB0 = rawA0 + 2 * TK * 128;
  auto rawA = [&](int b) { return rawA0 + (size_t)b * TK * 128; };
  auto rawB = [&](int b) { return rawB0 + (size_t)b * TK * 128; };
  const int nch = r0 < r1 ? (int)((r1 - r0 + TK - 1) / TK) : 0;
  auto prefetch = [&](int c, int b) {
    const int64_t rb = r0 + (int64_t)c * TK;
    const uint32_t rows = (uint32_t)(r1 - rb < TK ? r1 - rb : TK);
    const uint32_t ba = rows * P * 4u, bb = rows * Q * 4u;
    const uint8_t* ga = reinterpret_cast<const uint8_t*>(srcA + ((size_t)n * a.Bs + rb) * P);
    const uint8_t* gb = reinterpret_cast<const uint8_t*>(srcB + ((size_t)n * a.Bs + rb) * Q);
    uint8_t* da = reinterpret_cast<uint8_t*>(rawA(b));
    uint8_t* db = reinterpret_cast<uint8_t*>(rawB(b));
    mbar_expect_tx(&bars[1 + b], ba + bb);
    for (uint32_t o = 0; o < ba; o += 16384u) bulk_g2s(da + o, ga + o, min(16384u, ba - o), &bars[1 + b]);
    for (uint32_t o = 0; o < bb; o += 16384u) bulk_g2s(db + o, gb + o, min(16384u, bb - o), &bars[1 + b]);
  };
  if (t == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  // A image columns >= P stay 0 (M = 128 rows of the MMA)
  for (int e = t; e < (int)(2 * AB / 16); e += RT) reinterpret_cast<uint4*>(aimg)[e] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc(&tslot, 128);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  if (t == 0) {
    if (nch > 0) prefetch(0, 0);
    if (nch > 1) prefetch(1, 1);
  }
  const uint32_t idesc = idesc_bf16(128, Q, true, true);
  for (int c = 0; c < nch; ++c) {
    const int b = c & 1;
    const int64_t rb = r0 + (int64_t)c * TK;
    if (t < TK) {   // per-row scale of A: ā_{n+1} for dZ (which 2), 0 past the range
      const int64_t m = rb + t;
      srow[t] = m < r1 ? (which == 2 ? abar_of(a, n, m) : 1.0f) : 0.0f;
    }
    mbar_wait(&bars[1 + b], (uint32_t)((c >> 1) & 1));
    if (c > 0) mbar_wait(&bars[0], (uint32_t)((c - 1) & 1));   // MMA c-1 has read the images
    __syncthreads();
    const float* ra = rawA(b);
    const float* rbuf = rawB(b);
    const int pa = P / 4, qb = Q / 4;
    for (int e = t; e < TK * pa; e += RT) {
      const int rl = e / pa, c4 = 4 * (e - rl * pa);
      const float sc = srow[rl];
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (sc != 0.0f) {
        v = *reinterpret_cast<const float4*>(ra + rl * P + c4);
        v = make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w);
      }
      uint2 hi, lo;
      split4(v, hi, lo);
      *reinterpret_cast<uint2*>(aimg + ioff(rl, c4, 128)) = hi;
      *reinterpret_cast<uint2*>(aimg + AB + ioff(rl, c4, 128)) = lo;
    }
    for (int e = t; e < TK * qb; e += RT) {
      const int rl = e / qb, c4 = 4 * (e - rl * qb);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rb + rl < r1) v = *reinterpret_cast<const float4*>(rbuf + rl * Q + c4);
      uint2 hi, lo;
      split4(v, hi, lo);
      *reinterpret_cast<uint2*>(bimg + ioff(rl, c4, Q)) = hi;
      *reinterpret_cast<uint2*>(bimg + BB + ioff(rl, c4, Q)) = lo;
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (t == 0) {
      tc_after();
      if (c + 2 < nch) prefetch(c + 2, b);   // raw[b] consumed
      const Opnd Ah = mnmaj(aimg, 128), Al = mnmaj(aimg + AB, 128);
      const Opnd Bh = mnmaj(bimg, Q), Bl = mnmaj(bimg + BB, Q);
      gemm(tm, Ah, Bh, TK / 16, idesc, c > 0);
      gemm(tm, Ah, Bl, TK / 16, idesc, true);
      gemm(tm, Al, Bh, TK / 16, idesc, true);
      mma_commit(&bars[0]);
    }
  }
  if (nch > 0) {
    mbar_wait(&bars[0], (uint32_t)((nch - 1) & 1));
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

// Weight gradients from the tile images (compile-time shapes): one CTA per SM takes an
// equal share of the 3·N·2·tiles (which, step, 64-row half tile) units in order.  Thread
// 0 streams the four images of a unit (A hi / lo, B hi / lo: MN-major over the 64 rows,
// no conversion) by bulk copy into a ring of NSI stages, NSI - 1 units ahead, and issues
// the three MMA passes of each unit straight from its stage into the TMEM accumulator of
// the current (which, step) segment; all threads flush the segment with fp32 atomics.
// A rows past P (M = 128) read the neighbouring bytes of the stage: their products land
// in accumulator rows >= P, which the flush never reads.
constexpr int NSI = 3;
template <int WHICH>
__device__ __forceinline__ void tn_flush_img(const RowsArgs& a, int n, uint32_t tm) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int d = a.d, w = a.w;
  const int Q = WHICH == 0 ? a.Dp : a.Wp;
  const NetDims nd{d, w};
  float* G = a.grad + nd.step_base(n);
  const int qd = warp & 3, hh = warp >> 2, p = 32 * qd + lane;
  const uint32_t lb = tm + ((uint32_t)(32 * qd) << 16);
#pragma unroll 1
  for (int c0 = hh * (Q / 2); c0 < (hh + 1) * (Q / 2); c0 += 8) {
    uint32_t r8[8];
    tmem_ld8_nowait(lb + (uint32_t)c0, r8);
    tmem_ld_wait();
    reg_fence8(r8);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = c0 + e;
      const float v = __uint_as_float(r8[e]);
      if (v == 0.0f) continue;
      int64_t off = -1;
      if (WHICH == 0 && p < w) off = k < d ? nd.off_W1() + p * d + k : (k == d ? nd.off_b1() + p : -1);
      if (WHICH == 1 && p < w) off = k < w ? nd.off_W2() + p * w + k : (k == w ? nd.off_b2() + p : -1);
      if (WHICH == 2 && p < d) off = k < w ? nd.off_W3() + p * w + k : (k == w ? nd.off_b3() + p : -1);
      if (off >= 0) atomicAdd(G + off, v);
    }
  }
}
template <int DP, int WP>
__global__ void __launch_bounds__(RT, 1) k_rows_tn_img(RowsArgs a) {
  constexpr int KM = DP > WP ? DP : WP;
  constexpr uint32_t HB = 64u * KM * 2;              // one 64-row hi (or lo) image, max width
  constexpr uint32_t STB = 4 * HB;                   // stage: A hi, A lo, B hi, B lo
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NSI], mmab[NSI];
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  const int N = a.N;
  const int64_t nt2 = 2 * ((a.B + 127) / 128);        // 64-row units per (which, step)
  const int64_t U = 3LL * N * nt2;
  const int64_t u0 = blockIdx.x * U / gridDim.x, u1 = (blockIdx.x + 1) * U / gridDim.x;
  if (t == 0) {
    for (int i = 0; i < NSI; ++i) { mbar_init(&full[i], 1); mbar_init(&mmab[i], 1); }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 128);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = tslot;
  struct Cur { int which, n; int64_t k; };
  auto decode = [&](int64_t u) {
    const int64_t sgi = u / nt2;
    Cur c;
    c.k = u - sgi * nt2;
    c.which = (int)(sgi / N);
    c.n = (int)(sgi - (int64_t)c.which * N);
    return c;
  };
  auto advance = [&](Cur& c) {
    if (++c.k == nt2) { c.k = 0; if (++c.n == N) { c.n = 0; ++c.which; } }
  };
  auto issue_load = [&](const Cur& c, int stg) {   // thread 0
    const int P = c.which == 2 ? DP : WP, Q = c.which == 0 ? DP : WP;
    const float* srcA = c.which == 0 ? a.DA : c.which == 1 ? a.DH : a.GW;
    const float* srcB = c.which == 0 ? a.XT : c.which == 1 ? a.H1 : a.H2;
    const int64_t i0 = (c.k >> 1) * 128;
    const uint32_t half = (uint32_t)(c.k & 1);
    const uint8_t* ga = tile_img(srcA, a, c.n, i0, P) + half * 64u * P * 2;
    const uint8_t* gb = tile_img(srcB, a, c.n, i0, Q) + half * 64u * Q * 2;
    const uint32_t ba = 64u * P * 2, bb = 64u * Q * 2;   // <= 16 KB each
    uint8_t* st = sm + stg * STB;
    mbar_expect_tx(&full[stg], 2 * (ba + bb));
    bulk_g2s(st, ga, ba, &full[stg]);
    bulk_g2s(st + HB, ga + 128u * P * 2, ba, &full[stg]);
    bulk_g2s(st + 2 * HB, gb, bb, &full[stg]);
    bulk_g2s(st + 3 * HB, gb + 128u * Q * 2, bb, &full[stg]);
  };
  Cur cu = decode(u0 < U ? u0 : 0), cl = cu;
  if (t == 0)
    for (int i = 0; i < NSI && u0 + i < u1; ++i) { issue_load(cl, i); advance(cl); }
  bool seg_first = true;
  int stg = 0;
  uint32_t sph = 0;   // ring pass parity of stage stg
  for (int64_t u = u0, j = 0; u < u1; ++u, ++j) {
    const int which = cu.which, n = cu.n;
    const bool seg_end = u + 1 == u1 || cu.k + 1 == nt2;
    if (t == 0) {
      mbar_wait(&full[stg], sph);
      tc_after();
      const int P = which == 2 ? DP : WP, Q = which == 0 ? DP : WP;
      const uint32_t idesc = idesc_bf16(128, Q, true, true);
      uint8_t* st = sm + stg * STB;
      const Opnd Ah = mnmaj(st, P), Al = mnmaj(st + HB, P);
      const Opnd Bh = mnmaj(st + 2 * HB, Q), Bl = mnmaj(st + 3 * HB, Q);
      gemm(tm, Ah, Bh, 64 / 16, idesc, !seg_first);
      gemm(tm, Ah, Bl, 64 / 16, idesc, true);
      gemm(tm, Al, Bh, 64 / 16, idesc, true);
      mma_commit(&mmab[stg]);
      // refill the stage of the previous unit once its MMAs are done (NSI - 1 ahead)
      if (j > 0 && u - 1 + NSI < u1) {
        const int ps = stg == 0 ? NSI - 1 : stg - 1;
        const uint32_t pph = (stg == 0) ? (sph ^ 1u) : sph;
        mbar_wait(&mmab[ps], pph);
        issue_load(cl, ps);
        advance(cl);
      }
    }
    seg_first = false;
    if (seg_end) {   // flush the (which, step) accumulator
      // the other threads run ahead of thread 0 between flushes: they wait for this
      // unit's commit only once it is issued, so that the parity wait cannot alias an
      // earlier, still incomplete pass of the stage's barrier
      __syncthreads();
      mbar_wait(&mmab[stg], sph);
      tc_after();
      if (which == 0) tn_flush_img<0>(a, n, tm);
      else if (which == 1) tn_flush_img<1>(a, n, tm);
      else tn_flush_img<2>(a, n, tm);
      tc_before();
      __syncthreads();   // accumulator read before the next segment's first MMA
      seg_first = true;
    }
    advance(cu);
    if (++stg == NSI) { stg = 0; sph ^= 1u; }
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
template <int OP, int DP, int WP>
cudaError_t gemm_launch_t(const RowsArgs& a, cudaStream_t s) {
  constexpr int K = (OP == F1 || OP == B1) ? DP : WP, NC = (OP == F3) ? DP : WP;
  constexpr size_t half = 64 * (size_t)(NC + 4) * 4, ab2 = 2 * 128 * (size_t)K * 2;
  constexpr size_t smem = 2 * (size_t)NC * K * 2 + (half <= ab2 ? ab2 : ab2 + half);
  cudaError_t e = cudaFuncSetAttribute(k_rows_gemm_t<OP, DP, WP>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_rows_gemm_t<OP, DP, WP><<<dim3((unsigned)((a.B + 127) / 128), (unsigned)a.N), RT, smem, s>>>(a);
  return cudaGetLastError();
}

// compile-time shapes for the built (Dp, Wp) pairs, else the runtime-shaped kernel
#define BSDE_ROWS_SHAPES(X) X(112, 112) X(16, 32) X(48, 48) X(16, 16)

template <int OP>
cudaError_t gemm_launch(const RowsArgs& a, cudaStream_t s) {
  // compile-time shapes: F3 reads the H2 tile image; F1, F2, B1, B2 run inside the
  // fused kernels there (their buffers are tile images, which the unfused kernels
  // would misread)
#define X(DP_, WP_)                                                                       \
  if (a.Dp == DP_ && a.Wp == WP_)                                                        \
    return OP == F3 ? gemm_launch_t<F3, DP_, WP_>(a, s) : cudaErrorNotSupported;
  BSDE_ROWS_SHAPES(X)
#undef X
  const int K = (OP == F1 || OP == B1) ? a.Dp : a.Wp, Nc = (OP == F3) ? a.Dp : a.Wp;
  const size_t smem = 2 * (size_t)img_bytes(Nc, K) + 2 * (size_t)img_bytes(128, K) + 128 * (size_t)K * 4 +
                      128 * (size_t)(Nc + 4) * 4;
  cudaError_t e = cudaFuncSetAttribute(k_rows_gemm<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  // one CTA per SM over the N steps; each walks the row tiles of its step
  const int ntiles = (int)((a.B + 127) / 128), sms = sm_count();
  int g = (sms + a.N - 1) / a.N;
  if (g > ntiles) g = ntiles;
  if (g < 1) g = 1;
  k_rows_gemm<OP><<<dim3((unsigned)g, (unsigned)a.N), RT, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rows

bool rows_supported(int d, int w) { return d + 1 <= 128 && w + 1 <= 128; }

// compile-time shapes use the tile-image formats (row stride per step: whole tiles)
static bool rows_img_shape(int Dp, int Wp) {
#define X(DP_, WP_) if (Dp == DP_ && Wp == WP_) return true;
  BSDE_ROWS_SHAPES(X)
#undef X
  return false;
}
static int64_t rows_stride(int Dp, int Wp, int64_t B) {
  return rows_img_shape(Dp, Wp) ? (B + 127) / 128 * 128 : B;
}
size_t rows_buffer_bytes(int d, int w, int N, int64_t B) {
  const size_t Dp = rows::pad16(d + 1), Wp = rows::pad16(w + 1);
  const size_t R = (size_t)N * rows_stride((int)Dp, (int)Wp, B);
  return 4 * (2 * R * Dp + 4 * R * Wp + 2 * R + B) + 2 * 16 * R + 8 * 256;
}
size_t rows_pack_bytes(int d, int w, int N) {
  const int Dp = rows::pad16(d + 1), Wp = rows::pad16(w + 1);
  return (size_t)N * 2 * (rows::img_bytes(Wp, Dp) + rows::img_bytes(Wp, Wp) + rows::img_bytes(Dp, Wp));
}

// carve the row buffers [N_max][B] from base (rows_buffer_bytes)
void rows_carve(RowsArgs& a, void* base, int N_max) {
  a.Dp = rows::pad16(a.d + 1);
  a.Wp = rows::pad16(a.w + 1);
  a.Bs = rows_stride(a.Dp, a.Wp, a.B);
  uint8_t* p = static_cast<uint8_t*>(base);
  const size_t R = (size_t)N_max * a.Bs;
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
  a.M1 = reinterpret_cast<uint32_t*>(take(R * 4));
  a.M2 = reinterpret_cast<uint32_t*>(take(R * 4));
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
  rows::k_rows_paths<<<(unsigned)((a.B + rows::PPB - 1) / rows::PPB), rows::PPB * (a.Dp / 4), 0, s>>>(a);
  RCK(cudaGetLastError());
  bool fused = false;
#define X(DP_, WP_)                                                                               \
  if (a.Dp == DP_ && a.Wp == WP_) {   /* F1 + F2 fused: one CTA per SM over the steps */          \
    constexpr int KM_ = DP_ > WP_ ? DP_ : WP_;                                                     \
    const size_t smf = 2 * (size_t)WP_ * DP_ * 2 + 2 * (size_t)WP_ * WP_ * 2 + 2 * 128 * (size_t)KM_ * 2; \
    RCK(cudaFuncSetAttribute(rows::k_rows_f12_t<DP_, WP_>,                                         \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf));              \
    const int64_t nit = (int64_t)a.N * ((a.B + 127) / 128);   /* (step, tile) items */         \
    const int64_t sm_ = rows::sm_count();                                                                \
    const unsigned g = (unsigned)(nit < 1 ? 1 : (nit < sm_ ? nit : sm_));                       \
    rows::k_rows_f12_t<DP_, WP_><<<g, rows::RT, smf, s>>>(a);                                     \
    RCK(cudaGetLastError());                                                                       \
    fused = true;                                                                                  \
  }
  BSDE_ROWS_SHAPES(X)
#undef X
  if (!fused) {
    RCK(rows::gemm_launch<rows::F1>(a, s));
    RCK(rows::gemm_launch<rows::F2>(a, s));
  }
  RCK(rows::gemm_launch<rows::F3>(a, s));
  rows::k_rows_y<<<(unsigned)((a.B + 255) / 256), 256, 0, s>>>(a);
  RCK(cudaGetLastError());
  if (launches) *launches += fused ? 4 : 5;
  return cudaSuccess;
}

// adjoint: B1, B2 and the three weight-gradient GEMMs (one launch)
cudaError_t launch_rows_backward(const RowsArgs& a, cudaStream_t s, int* launches) {
  const int sms = rows::sm_count();
  bool fused = false;
#define X(DP_, WP_)                                                                               \
  if (a.Dp == DP_ && a.Wp == WP_) {   /* B1 + B2 fused: one CTA per SM over the steps */          \
    constexpr int KM_ = DP_ > WP_ ? DP_ : WP_;                                                     \
    const size_t smb = 2 * (size_t)DP_ * WP_ * 2 + 2 * (size_t)WP_ * WP_ * 2 + 2 * 128 * (size_t)KM_ * 2; \
    RCK(cudaFuncSetAttribute(rows::k_rows_b12_t<DP_, WP_>,                                         \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));              \
    const int64_t nit = (int64_t)a.N * ((a.B + 127) / 128);   /* (step, tile) items */         \
    const int64_t sm_ = sms;                                                                \
    const unsigned g = (unsigned)(nit < 1 ? 1 : (nit < sm_ ? nit : sm_));                       \
    rows::k_rows_b12_t<DP_, WP_><<<g, rows::RT, smb, s>>>(a);                                     \
    RCK(cudaGetLastError());                                                                       \
    fused = true;                                                                                  \
  }
  BSDE_ROWS_SHAPES(X)
#undef X
  if (!fused) {
    RCK(rows::gemm_launch<rows::B1>(a, s));
    RCK(rows::gemm_launch<rows::B2>(a, s));
  }
#define X(DP_, WP_)                                                                               \
  if (a.Dp == DP_ && a.Wp == WP_) {   /* compile-time shapes: tile images, one CTA per SM */      \
    constexpr int KM_ = DP_ > WP_ ? DP_ : WP_;                                                     \
    const size_t smt = rows::NSI * 4 * 64 * (size_t)KM_ * 2;                                      \
    RCK(cudaFuncSetAttribute(rows::k_rows_tn_img<DP_, WP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smt));                                                           \
    rows::k_rows_tn_img<DP_, WP_><<<sms, rows::RT, smt, s>>>(a);                                   \
    RCK(cudaGetLastError());                                                                       \
    if (launches) *launches += fused ? 2 : 3;                                                      \
    return cudaSuccess;                                                                            \
  }
  BSDE_ROWS_SHAPES(X)
#undef X
  // one CTA per SM over the 3·N weight-gradient problems, >= 256 rows each
  int split = (int)((sms + 3LL * a.N - 1) / (3LL * a.N));
  const int64_t maxsplit = (a.B + 255) / 256;
  if (split > maxsplit) split = (int)maxsplit;
  if (split < 1) split = 1;
  const int rpc = (int)((a.B + split - 1) / split);
  const size_t smem = 2 * (size_t)rows::img_bytes(rows::TK, 128) + 2 * (size_t)rows::img_bytes(rows::TK, 128) +
                      4 * (size_t)rows::TK * 128 * 4;
  RCK(cudaFuncSetAttribute(rows::k_rows_tn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  rows::k_rows_tn<<<dim3((unsigned)((a.B + rpc - 1) / rpc), 3, (unsigned)a.N), rows::RT, smem, s>>>(a, rpc);
  RCK(cudaGetLastError());
  if (launches) *launches += 3;
  return cudaSuccess;
}

}  // namespace bsde
