// tc.cu — tcgen05 (sm_100a) forward and adjoint kernels: bf16 operands in shared
// memory, fp32 accumulators in tensor memory (TMEM), one CTA of 512 threads per SM.
//
// Thread layout: warp w accesses TMEM lanes 32·(w%4)..+31, so a 128-path tile is
// one path per lane and four threads per path; thread group g = w/4 owns the
// 8-column chunks g, g+4, g+8, g+12 of every 112-column accumulator / operand
// image (loads: 4 × tcgen05.ld.32x32b.x8 and one wait).
//
// Data flow:
//  k_pack_tc  fp32 master θ -> per-step bf16 operand images W̃1 [Wp×Dp], W̃2 [Wp×Wp],
//             W̃3 [Dp×Wp] with the biases folded into a constant-1 column
//             (W̃1 row w = e_d makes H1[w] = 1; W̃2/W̃3 take b2/b3 in column w).
//  k_fwd_tc   tile-major: one 128-path tile walks all N steps: a1 Philox ΔW (computed
//             while the step's GEMMs run), a2 Euler X (fp32 registers), a3 three
//             tcgen05 GEMMs (weights double-buffered by bulk copy), a4 Y update, a5
//             terminal loss; each X_n operand image is bulk-copied to HBM for the
//             adjoint pass.
//  k_bwd_tc   step-major: each CTA owns a contiguous range of (n, tile) items,
//             recomputes the step-n net, forms dZ_n = ā_{n+1}(ΔW_n - Δt ∂_z f),
//             back-propagates with 2 input-gradient GEMMs and accumulates the 3
//             weight-gradient GEMMs (contracting over paths, MN-major operands) in
//             TMEM across its range; one flush of fp32 atomics per step change.
//
// Citations: Eq. 5, Eq. 7, Eq. 6.
#include "kernels.cuh"
#include "tc_common.cuh"

namespace bsde {
namespace tc {

constexpr int NTH = 512;   // threads per CTA (4 per path)
template <int D>
constexpr int kDwChunks = (D + 7) / 8;   // 8-column chunks of the stored ΔW image
constexpr float kSqrt2 = 1.41421356237309515f;

// ------------------------------------------------------------------ weight packing
template <int D, int W>
__global__ void k_pack_tc(const float* __restrict__ params, uint8_t* __restrict__ out, int N) {
  using Dm = Dims<D, W>;
  const NetDims nd{D, W};
  constexpr int c1 = Dm::Wp * (Dm::Dp / 8), c2 = Dm::Wp * (Dm::Wp / 8), c3 = Dm::Dp * (Dm::Wp / 8);
  constexpr int per_step = c1 + c2 + c3;
  const int64_t total = (int64_t)N * per_step;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / per_step);
    int r = (int)(i - (int64_t)n * per_step);
    const float* P = params + nd.step_base(n);
    uint8_t* img = out + (size_t)n * Dm::WB;
    float v[8];
    int row, chunk, C;
    if (r < c1) {                       // W̃1 [Wp × Dp]: [W1 | b1], row W = e_D
      C = Dm::Dp; row = r / (C / 8); chunk = r - row * (C / 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = chunk * 8 + e;
        float x = 0.0f;
        if (row < W) x = k < D ? P[nd.off_W1() + row * D + k] : (k == D ? P[nd.off_b1() + row] : 0.0f);
        else if (row == W) x = (k == D) ? 1.0f : 0.0f;
        v[e] = x;
      }
    } else if (r < c1 + c2) {           // W̃2 [Wp × Wp]: [W2 | b2], rows >= W zero
      r -= c1; img += Dm::W1B;
      C = Dm::Wp; row = r / (C / 8); chunk = r - row * (C / 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = chunk * 8 + e;
        float x = 0.0f;
        if (row < W) x = k < W ? P[nd.off_W2() + row * W + k] : (k == W ? P[nd.off_b2() + row] : 0.0f);
        v[e] = x;
      }
    } else {                            // W̃3 [Dp × Wp]: [W3 | b3], rows >= D zero
      r -= c1 + c2; img += Dm::W1B + Dm::W2B;
      C = Dm::Wp; row = r / (C / 8); chunk = r - row * (C / 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = chunk * 8 + e;
        float x = 0.0f;
        if (row < D) x = k < W ? P[nd.off_W3() + row * W + k] : (k == W ? P[nd.off_b3() + row] : 0.0f);
        v[e] = x;
      }
    }
    st_chunk(img, row, chunk, C, v);
  }
}

// Column predicates of this thread's chunks c = g + 4i (g = 0..3) that fold at
// compile time after unrolling: column 8(g+4i)+e is < LIM for every g when
// 8(3+4i)+e < LIM, and for no g when 8(4i)+e >= LIM.
__device__ __forceinline__ bool col_lt(int g, int i, int e, int LIM) {
  return (8 * (3 + 4 * i) + e < LIM) || (8 * (4 * i) + e < LIM && 8 * (g + 4 * i) + e < LIM);
}
// chunk g + 4i exists in an image of NC chunks
__device__ __forceinline__ bool chunk_lt(int g, int i, int NC) {
  return (3 + 4 * i < NC) || (4 * i < NC && g + 4 * i < NC);
}

// ΔW_n at this thread's columns, dw[8i + e] = ΔW[8(g + 4i) + e] (columns < D),
// produced one Philox block (4 normals) per call so that the generation can fill
// the waits for the tensor core ("work while waiting").
struct DwGen {
  uint32_t m, n, it, k0, k1;
  float sdt;
  int g;   // slot s = (i, h) = (s/2, s%2) holds 4-block 2(g+4i)+h
  // slots [S0, S1) — a compile-time share of the step's RNG, issued right after
  // a GEMM so that the generation overlaps it
  // The Philox rounds of all slots are interleaved (independent dependency chains
  // give the scheduler ILP), then the Box-Muller maps.  Slots whose columns are
  // >= D for every column group are skipped at compile time.
  template <int D, int S0, int S1>
  __device__ __forceinline__ void run(float (&dw)[32]) const {
    constexpr int K = S1 - S0;
    uint4 c[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int s = S0 + j;
      c[j] = make_uint4((uint32_t)(2 * (g + 4 * (s / 2)) + s % 2), m, n, it);
    }
    uint32_t a0 = k0, a1 = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r) { a0 += kPhiloxW0; a1 += kPhiloxW1; }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int s = S0 + j;
        if (8 * (4 * (s / 2)) + 4 * (s % 2) >= D) continue;   // never valid
        const uint32_t lo0 = kPhiloxM0 * c[j].x, hi0 = __umulhi(kPhiloxM0, c[j].x);
        const uint32_t lo1 = kPhiloxM1 * c[j].z, hi1 = __umulhi(kPhiloxM1, c[j].z);
        c[j] = make_uint4(hi1 ^ c[j].y ^ a0, lo1, hi0 ^ c[j].w ^ a1, lo0);
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int s = S0 + j, i = s / 2, h = s % 2;
      float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
      if (8 * (4 * i) + 4 * h < D) {
        box_muller_fast(c[j].x, c[j].y, sdt, z0, z1);
        box_muller_fast(c[j].z, c[j].w, sdt, z2, z3);
      }
      const bool ok = col_lt(g, i, 4 * h, D);
      dw[8 * i + 4 * h + 0] = ok ? z0 : 0.f;
      dw[8 * i + 4 * h + 1] = ok ? z1 : 0.f;
      dw[8 * i + 4 * h + 2] = ok ? z2 : 0.f;
      dw[8 * i + 4 * h + 3] = ok ? z3 : 0.f;
    }
  }
};

// ------------------------------------------------------------------ forward
template <int D, int W>
__global__ void __launch_bounds__(NTH, 1) k_fwd_tc(PassArgs a, int ntiles) {
  using Dm = Dims<D, W>;
  constexpr int Dp = Dm::Dp, Wp = Dm::Wp;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* wimg0 = sm;
  uint8_t* wimg1 = sm + Dm::WB;
  uint8_t* xop = sm + 2 * Dm::WB;
  uint8_t* hop = xop + Dm::ACT;
  float2* red = reinterpret_cast<float2*>(hop + Dm::ACT);            // [2][4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 8 * 128);       // [0],[1] weights, [2] mma
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  __shared__ double lred[4];
  __shared__ float gred[4];

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int q = warp & 3, g = warp >> 2;
  const int row = 32 * q + lane;
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = *tslot;
  const uint32_t lq = ((uint32_t)(32 * q) << 16) + 8u * g;   // lane quadrant + first chunk column
  const uint32_t acc0 = tm + lq, acc1 = tm + 128 + lq;

  const int N = a.N;
  const uint8_t* wsrc = static_cast<const uint8_t*>(a.wpack);
  uint8_t* xst = static_cast<uint8_t*>(a.xpack);
  const uint32_t it = a.eval ? a.eval_it : a.state->it;
  const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int64_t total_seq = (int64_t)my_tiles * N;
  constexpr uint32_t I1 = idesc_bf16(128, Wp, false, false);
  constexpr uint32_t I3 = idesc_bf16(128, Dp, false, false);

  auto load_weights = [&](int64_t s) {   // thread 0
    const int n = (int)(s % N);
    uint8_t* dst = (s & 1) ? wimg1 : wimg0;
    uint64_t* bar = &bars[s & 1];
    mbar_expect_tx(bar, Dm::WB);
    const uint8_t* src = wsrc + (size_t)n * Dm::WB;
    for (uint32_t off = 0; off < Dm::WB; off += 16384u)
      bulk_g2s(dst + off, src + off, min(16384u, Dm::WB - off), bar);
  };
  if (t == 0 && total_seq > 0) load_weights(0);

  // debug trace: thread 32 of CTA 0 stamps clock64() at the phase boundaries of its steps
  unsigned long long* const clk = (a.clk && blockIdx.x == 0 && t == 32) ? a.clk : nullptr;
#define CLK(i) do { if (clk && s < 64) clk[s * 16 + (i)] = clock64(); } while (0)
  uint32_t mph = 0;
  int64_t s = 0;
  double lsum = 0.0;
  float dy0 = 0.0f;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t mloc = (int64_t)tile * 128 + row;
    const bool valid = mloc < a.B_local;
    const uint32_t mg = (uint32_t)(a.m0 + mloc);
    float X[32];                       // X at this thread's columns
#pragma unroll
    for (int i = 0; i < 32; ++i) X[i] = a.x0;
    float Y = a.params[0];
    for (int n = 0; n < N; ++n, ++s) {
      uint8_t* wimg = (s & 1) ? wimg1 : wimg0;
      CLK(0);
      if (t == 0 && s + 1 < total_seq) load_weights(s + 1);
      // X_n operand chunks (bf16; column D is the constant 1 of the folded bias)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (chunk_lt(g, i, Dp / 8)) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = 8 * (g + 4 * i) + e;
            v[e] = col_lt(g, i, e, D) ? X[8 * i + e] : (j == D ? 1.0f : 0.0f);
          }
          st_chunk(xop, row, g + 4 * i, Dp, v);
        }
      }
      fence_async_smem();
      CLK(1);
      __syncthreads();
      CLK(2);
      if (n > 0) {   // finish a4 of step n-1 from the partial sums of the four threads
        const float2 r0 = red[row], r1 = red[128 + row], r2 = red[256 + row], r3 = red[384 + row];
        const float cz = (r0.x + r1.x) + (r2.x + r3.x), zz = (r0.y + r1.y) + (r2.y + r3.y);
        Y = Y - driver_f(a.problem, Y, zz, a.lam) * a.dt + cz;
      }
      if (!a.eval && a.problem == kAllenCahn && valid && g == 0)
        a.Ystore[(int64_t)n * a.B_local + mloc] = Y;
      if (t == 0) {
        if (!a.eval) {
          bulk_s2g(xst + ((size_t)n * ntiles + tile) * Dm::XB, xop, Dm::XB);
          bulk_commit();
        }
        mbar_wait(&bars[s & 1], (uint32_t)((s >> 1) & 1));
        tc_after();
        gemm(tm, kmaj(xop, Dp), kmaj(wimg, Dp), Dp / 16, I1, false);                  // A1
        mma_commit(&bars[2]);
      }
      float dw[32];                                // a1: ΔW_n, generated while the GEMMs run
      const DwGen gen{mg, (uint32_t)n, it, a.k0, a.k1, a.sqrt_dt, g};
      gen.run<D, 0, 4>(dw);
      CLK(3);
      mbar_wait(&bars[2], mph);
      mph ^= 1;
      CLK(4);
      tc_after();
      {  // H1 = ReLU(A1)
        float v[32];
        tmem_ld4x8(acc0, v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (chunk_lt(g, i, Wp / 8)) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[8 * i + e] = fmaxf(v[8 * i + e], 0.0f);
            st_chunk(hop, row, g + 4 * i, Wp, v + 8 * i);
          }
        }
      }
      fence_async_smem();
      tc_before();
      CLK(5);
      __syncthreads();
      CLK(6);
      if (t == 0) {
        tc_after();
        gemm(tm + 128, kmaj(hop, Wp), kmaj(wimg + Dm::W1B, Wp), Wp / 16, I1, false);   // A2
        mma_commit(&bars[2]);
      }
      gen.run<D, 4, 8>(dw);
      CLK(7);
      mbar_wait(&bars[2], mph);
      mph ^= 1;
      CLK(8);
      tc_after();
      {  // H2 = ReLU(A1) + ReLU(A2) (residual block, Eq. 7 with h = 1), over H1 in hop
        float v1[32], v2[32];
        tmem_ld4x8(acc0, v1);
        tmem_ld4x8(acc1, v2);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (chunk_lt(g, i, Wp / 8)) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              v1[8 * i + e] = fmaxf(v1[8 * i + e], 0.0f) + fmaxf(v2[8 * i + e], 0.0f);
            st_chunk(hop, row, g + 4 * i, Wp, v1 + 8 * i);
          }
        }
      }
      fence_async_smem();
      tc_before();
      if (t == 0 && !a.eval) bulk_wait_read0();   // the X_n image has left xop
      CLK(9);
      __syncthreads();
      CLK(10);
      if (t == 0) {
        tc_after();
        gemm(tm, kmaj(hop, Wp), kmaj(wimg + Dm::W1B + Dm::W2B, Wp), Wp / 16, I3, false);  // Z
        mma_commit(&bars[2]);
      }
      // (all ΔW slots generated during G1 and G2)
      CLK(11);
      mbar_wait(&bars[2], mph);
      mph ^= 1;
      CLK(12);
      tc_after();
      float cz = 0.0f, zz = 0.0f;
      {  // a4 partials c = Z·ΔW, |Z|²; a2: X += √2 ΔW
        float z[32];
        tmem_ld4x8(acc0, z);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if (col_lt(g, i, e, D)) {
              cz = fmaf(z[8 * i + e], dw[8 * i + e], cz);
              zz = fmaf(z[8 * i + e], z[8 * i + e], zz);
              X[8 * i + e] = fmaf(kSqrt2, dw[8 * i + e], X[8 * i + e]);
            }
          }
        }
      }
      red[g * 128 + row] = make_float2(cz, zz);   // a4 is finished at the next step's barrier
      CLK(13);
      tc_before();
    }
    // a5: R = Y_N - g(X_N); loss; ā recursion and dY0
    float sx = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (col_lt(g, i, e, D)) sx = fmaf(X[8 * i + e], X[8 * i + e], sx);
    red[512 + g * 128 + row] = make_float2(sx, 0.0f);
    __syncthreads();
    {
      const float2 r0 = red[row], r1 = red[128 + row], r2 = red[256 + row], r3 = red[384 + row];
      const float cz = (r0.x + r1.x) + (r2.x + r3.x), zz = (r0.y + r1.y) + (r2.y + r3.y);
      Y = Y - driver_f(a.problem, Y, zz, a.lam) * a.dt + cz;                         // a4, n = N-1
    }
    sx = (red[512 + row].x + red[640 + row].x) + (red[768 + row].x + red[896 + row].x);
    __syncthreads();   // red is rewritten by the next tile's first step
    if (g == 0 && valid) {
      const float R = Y - terminal_g(a.problem, sx);
      lsum += (double)R * R;
      if (!a.eval) {
        a.Rstore[mloc] = R;
        float ab = 2.0f * R * a.inv_B;
        if (a.problem == kAllenCahn) {
          for (int n = N - 1; n >= 0; --n) {
            const float y = a.Ystore[(int64_t)n * a.B_local + mloc];
            a.abar[(int64_t)n * a.B_local + mloc] = ab;               // ā_{n+1}
            ab *= 1.0f - a.dt * driver_dfdy(a.problem, y);
          }
        } else {
          a.abar[mloc] = ab;                                          // ā_N
        }
        dy0 += ab;
      }
    }
  }
  double lw = lsum;
  float gw = dy0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lw += __shfl_xor_sync(0xffffffffu, lw, o);
    gw += __shfl_xor_sync(0xffffffffu, gw, o);
  }
  if (g == 0 && lane == 0) { lred[q] = lw; gred[q] = gw; }
  tc_before();
  __syncthreads();
  if (t == 0) {
    const double L = lred[0] + lred[1] + lred[2] + lred[3];
    if (L != 0.0) atomicAdd(a.loss_acc, L);
    const float g0 = gred[0] + gred[1] + gred[2] + gred[3];
    if (!a.eval && g0 != 0.0f) atomicAdd(a.grad, g0);
    if (!a.eval) bulk_wait0();
  }
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 256);
  }
#undef CLK
}

// ------------------------------------------------------------------ adjoint
template <int D, int W>
__global__ void __launch_bounds__(NTH, 1) k_bwd_tc(PassArgs a, int ntiles, int64_t items) {
  using Dm = Dims<D, W>;
  constexpr int Dp = Dm::Dp, Wp = Dm::Wp;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* wimg = sm;
  uint8_t* xbuf0 = sm + Dm::WB;
  uint8_t* xbuf1 = xbuf0 + Dm::ACT;
  uint8_t* hop = xbuf1 + Dm::ACT;     // H1
  uint8_t* b2 = hop + Dm::ACT;        // H2, then dA2
  uint8_t* b3 = b2 + Dm::ACT;         // dZ, then dA1
  // barriers: 0 weights, 1-2 X images, 3 chain MMAs, 4 G8, 5 G5, 6 G7
  uint64_t* bars = reinterpret_cast<uint64_t*>(b3 + Dm::ACT);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int q = warp & 3, g = warp >> 2;
  const int row = 32 * q + lane;
  if (t == 0) {
    for (int i = 0; i < 7; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = *tslot;
  const uint32_t lq = ((uint32_t)(32 * q) << 16) + 8u * g;
  const uint32_t acc = tm, G1 = tm + 128, G2 = tm + 256, G3 = tm + 384;

  const int64_t i0 = blockIdx.x * items / gridDim.x, i1 = (blockIdx.x + 1) * items / gridDim.x;
  const uint8_t* wsrc = static_cast<const uint8_t*>(a.wpack);
  const uint8_t* xst = static_cast<const uint8_t*>(a.xpack);
  const uint32_t it = a.state->it;
  const NetDims nd{D, W};
  const float zc = -a.dt * driver_dfdz_coef(a.problem, a.lam);
  constexpr uint32_t IW = idesc_bf16(128, Wp, false, false);     // G1, G2
  constexpr uint32_t ID = idesc_bf16(128, Dp, false, false);     // G3
  constexpr uint32_t IWm = idesc_bf16(128, Wp, false, true);     // G4, G6 (B = W̃ᵀ view)
  constexpr uint32_t IGW = idesc_bf16(128, Wp, true, true);      // G5, G7 (over paths)
  constexpr uint32_t IGD = idesc_bf16(128, Dp, true, true);      // G8

  auto load_x = [&](int64_t item) {   // thread 0
    const int buf = (int)((item - i0) & 1);
    const int n = (int)(item / ntiles), tile = (int)(item - (int64_t)n * ntiles);
    uint64_t* bar = &bars[1 + buf];
    mbar_expect_tx(bar, Dm::XB);
    bulk_g2s(buf ? xbuf1 : xbuf0, xst + ((size_t)n * ntiles + tile) * Dm::XB, Dm::XB, bar);
  };
  if (t == 0) {
    if (i0 < i1) load_x(i0);
    if (i0 + 1 < i1) load_x(i0 + 1);
  }

  uint32_t mph = 0, wph = 0, gph = 0, g5ph = 0, g7ph = 0;
  unsigned long long* const clk = (a.clk && blockIdx.x == 0 && t == 32) ? a.clk : nullptr;
#define CLK(i) do { if (clk && item - i0 < 64) clk[(item - i0) * 16 + (i)] = clock64(); } while (0)
  int cur_n = -1;
  bool first = true;
  bool g8_pending = false;

  // gradient flush of step cur_n: TMEM -> fp32 atomics (lane = gradient row,
  // this thread's column chunks)
  auto flush = [&]() {
    if (g8_pending) {            // G7 and G8 of the last item
      mbar_wait(&bars[6], g7ph);
      g7ph ^= 1;
      mbar_wait(&bars[4], gph);
      gph ^= 1;
      g8_pending = false;
    }
    tc_after();
    float* G = a.grad + nd.step_base(cur_n);
    float v[32];
    tmem_ld4x8(G1 + lq, v);                          // dW̃1 row = w-unit, cols = d-inputs
    if (row < W) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int k = 8 * (g + 4 * (i / 8)) + (i % 8);
        if (k < D) atomicAdd(G + nd.off_W1() + row * D + k, v[i]);
        else if (k == D) atomicAdd(G + nd.off_b1() + row, v[i]);
      }
    }
    tmem_ld4x8(G2 + lq, v);                          // dW̃2
    if (row < W) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int k = 8 * (g + 4 * (i / 8)) + (i % 8);
        if (k < W) atomicAdd(G + nd.off_W2() + row * W + k, v[i]);
        else if (k == W) atomicAdd(G + nd.off_b2() + row, v[i]);
      }
    }
    tmem_ld4x8(G3 + lq, v);                          // dW̃3 row = d-output
    if (row < D) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int k = 8 * (g + 4 * (i / 8)) + (i % 8);
        if (k < W) atomicAdd(G + nd.off_W3() + row * W + k, v[i]);
        else if (k == W) atomicAdd(G + nd.off_b3() + row, v[i]);
      }
    }
    tc_before();
    __syncthreads();
  };

  for (int64_t item = i0; item < i1; ++item) {
    const int n = (int)(item / ntiles), tile = (int)(item - (int64_t)n * ntiles);
    const int buf = (int)((item - i0) & 1);
    uint8_t* xop = buf ? xbuf1 : xbuf0;
    if (n != cur_n) {
      if (cur_n >= 0) flush();
      if (t == 0) {
        mbar_expect_tx(&bars[0], Dm::WB);
        const uint8_t* src = wsrc + (size_t)n * Dm::WB;
        for (uint32_t off = 0; off < Dm::WB; off += 16384u)
          bulk_g2s(wimg + off, src + off, min(16384u, Dm::WB - off), &bars[0]);
      }
      mbar_wait(&bars[0], wph);
      wph ^= 1;
      cur_n = n;
      first = true;
    }
    CLK(0);
    const int64_t mloc = (int64_t)tile * 128 + row;
    const bool valid = mloc < a.B_local;
    const uint32_t mg = (uint32_t)(a.m0 + mloc);
    const float ab = valid ? (a.problem == kAllenCahn ? a.abar[(int64_t)n * a.B_local + mloc]
                                                      : a.abar[mloc])
                           : 0.0f;
    if (t == 0) {   // G1: A1 = X̃ W̃1ᵀ (recompute)
      mbar_wait(&bars[1 + buf], (uint32_t)(((item - i0) >> 1) & 1));
      tc_after();
      gemm(acc, kmaj(xop, Dp), kmaj(wimg, Dp), Dp / 16, IW, false);
      mma_commit(&bars[3]);
    }
    float dw[32];   // ΔW_n regenerated (Philox) while G1..G3 run
    const DwGen gen{mg, (uint32_t)n, it, a.k0, a.k1, a.sqrt_dt, g};
    gen.run<D, 0, 4>(dw);
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(1);
    if (g8_pending) {            // the previous item's G7, G8 were issued before G1
      mbar_wait(&bars[6], g7ph);
      g7ph ^= 1;
      mbar_wait(&bars[4], gph);
      gph ^= 1;
      g8_pending = false;
    }
    if (t == 0 && item + 1 < i1 && item > i0) load_x(item + 1);   // its buffer's last reader (G8) is done
    tc_after();
    uint32_t m1 = 0, m2 = 0;   // ReLU masks of this thread's 32 columns
    {
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (v[i] > 0.0f) m1 |= 1u << i;
        v[i] = fmaxf(v[i], 0.0f);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Wp / 8))st_chunk(hop, row, g + 4 * i, Wp, v + 8 * i);
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    CLK(2);
    if (t == 0) {   // G2: A2 = H1 W̃2ᵀ
      tc_after();
      gemm(acc, kmaj(hop, Wp), kmaj(wimg + Dm::W1B, Wp), Wp / 16, IW, false);
      mma_commit(&bars[3]);
    }
    gen.run<D, 4, 8>(dw);
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(3);
    tc_after();
    {  // H2 = H1 (bf16 copy, R17) + ReLU(A2), chunk by chunk
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (v[i] > 0.0f) m2 |= 1u << i;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Wp / 8)) {
          float h[8];
          ld_chunk(hop, row, g + 4 * i, Wp, h);
#pragma unroll
          for (int e = 0; e < 8; ++e) h[e] += fmaxf(v[8 * i + e], 0.0f);
          st_chunk(b2, row, g + 4 * i, Wp, h);
        }
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    CLK(4);
    if (t == 0) {   // G3: Z = H2 W̃3ᵀ
      tc_after();
      gemm(acc, kmaj(b2, Wp), kmaj(wimg + Dm::W1B + Dm::W2B, Wp), Wp / 16, ID, false);
      mma_commit(&bars[3]);
    }
    // (all ΔW slots generated during G1 and G2)
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(5);
    tc_after();
    {  // dZ = ā_{n+1}(ΔW_n - Δt ∂_z f), columns >= D zero
      float z[32];
      tmem_ld4x8(acc + lq, z);
#pragma unroll
      for (int i = 0; i < 32; ++i)
        z[i] = col_lt(g, i / 8, i % 8, D) ? ab * fmaf(zc, z[i], dw[i]) : 0.0f;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Dp / 8)) st_chunk(b3, row, g + 4 * i, Dp, z + 8 * i);
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    CLK(6);
    if (t == 0) {
      tc_after();
      // G4: dH2 = dZ W̃3 ; G5: dW̃3 += dZᵀ H2
      gemm(acc, kmaj(b3, Dp), mnmaj(wimg + Dm::W1B + Dm::W2B, Wp), Dp / 16, IWm, false);
      mma_commit(&bars[3]);
      gemm(G3, mnmaj(b3, Dp), mnmaj(b2, Wp), 128 / 16, IGW, !first);
      mma_commit(&bars[5]);
    }
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(7);
    tc_after();
    {  // dA2 = dH2 ⊙ 1[A2 > 0]  (computed while G5 runs; stored over H2 once G5 is done)
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = (m2 >> i) & 1u ? v[i] : 0.0f;
      mbar_wait(&bars[5], g5ph);
      g5ph ^= 1;
      CLK(8);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Wp / 8))st_chunk(b2, row, g + 4 * i, Wp, v + 8 * i);
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    CLK(9);
    if (t == 0) {
      tc_after();
      // G6: dH1 = dH2 + dA2 W̃2 (accumulated onto dH2) ; G7: dW̃2 += dA2ᵀ H1
      gemm(acc, kmaj(b2, Wp), mnmaj(wimg + Dm::W1B, Wp), Wp / 16, IWm, true);
      mma_commit(&bars[3]);
      gemm(G2, mnmaj(b2, Wp), mnmaj(hop, Wp), 128 / 16, IGW, !first);
      mma_commit(&bars[6]);
    }
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(10);
    tc_after();
    {  // dA1 = dH1 ⊙ 1[A1 > 0]
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = (m1 >> i) & 1u ? v[i] : 0.0f;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Wp / 8))st_chunk(b3, row, g + 4 * i, Wp, v + 8 * i);
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    CLK(11);
    if (t == 0) {   // G8: dW̃1 += dA1ᵀ X̃
      tc_after();
      gemm(G1, mnmaj(b3, Wp), mnmaj(xop, Dp), 128 / 16, IGD, !first);
      mma_commit(&bars[4]);
    }
    g8_pending = true;
    first = false;
    CLK(12);
  }
  if (cur_n >= 0) flush();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 512);
  }
#undef CLK
}

// ------------------------------------------------------------------ UMMA self-test
// mode 0: D = A·Bᵀ, A [128×112] and B [112×112] K-major (like the forward GEMMs)
// mode 1: D = A·B,  A [128×112] K-major, B [112(k)×112(n)] MN-major view (like G4/G6)
// mode 2: D = Aᵀ·B, A [128(k)×112(m)], B [128(k)×112(n)], both MN-major (like G5/G7/G8);
//         output rows m >= 112 are undefined.
__global__ void __launch_bounds__(128, 1) k_umma_test(int mode, const float* A, const float* B,
                                                      float* Dout) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int C = 112;
  uint8_t* aimg = sm;
  uint8_t* bimg = sm + 128 * C * 2 + 256;
  uint64_t* bar = reinterpret_cast<uint64_t*>(bimg + 128 * C * 2 + 256);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int t = threadIdx.x, warp = t >> 5;
  const int brows = mode == 2 ? 128 : 112;
  for (int r = 0; r < 128; ++r)
    if (t < C / 8) {
      float v[8];
      for (int e = 0; e < 8; ++e) v[e] = A[r * C + t * 8 + e];
      st_chunk(aimg, r, t, C, v);
    }
  for (int r = 0; r < brows; ++r)
    if (t < C / 8) {
      float v[8];
      for (int e = 0; e < 8; ++e) v[e] = B[r * C + t * 8 + e];
      st_chunk(bimg, r, t, C, v);
    }
  if (t == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(tslot, 128);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = *tslot;
  if (t == 0) {
    if (mode == 0) gemm(tm, kmaj(aimg, C), kmaj(bimg, C), C / 16, idesc_bf16(128, 112, false, false), false);
    if (mode == 1) gemm(tm, kmaj(aimg, C), mnmaj(bimg, C), C / 16, idesc_bf16(128, 112, false, true), false);
    if (mode == 2) gemm(tm, mnmaj(aimg, C), mnmaj(bimg, C), 128 / 16, idesc_bf16(128, 112, true, true), false);
    mma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_after();
  for (int c = 0; c < C / 16; ++c) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + c * 16, v);
    for (int e = 0; e < 16; ++e) Dout[t * C + c * 16 + e] = v[e];
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 128);
  }
}

__global__ void k_debug_dw_fast(uint32_t it, int n, int64_t m0, int64_t count, int d, float sdt,
                                uint32_t k0, uint32_t k1, float* out) {
  const int nq = (d + 3) >> 2;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count * nq) return;
  const int64_t p = i / nq;
  const int q = (int)(i - p * nq);
  const float4 z = dw4_fast((uint32_t)q, (uint32_t)(m0 + p), (uint32_t)n, it, k0, k1, sdt);
  const float zz[4] = {z.x, z.y, z.z, z.w};
  for (int k = 0; k < 4; ++k)
    if (4 * q + k < d) out[p * d + 4 * q + k] = zz[k];
}

// ------------------------------------------------------------------ dispatch
template <int D, int W>
struct Impl {
  using Dm = Dims<D, W>;
  static size_t fwd_smem() { return 2 * Dm::WB + 2 * Dm::ACT + 8 * 128 * 8 + 64; }
  static size_t bwd_smem() { return Dm::WB + 5 * Dm::ACT + 96; }
  static int ntiles(const PassArgs& a) { return (int)((a.B_local + 127) / 128); }
  static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }
  static cudaError_t fwd(const PassArgs& a, cudaStream_t s) {
    const size_t smem = fwd_smem();
    cudaError_t e = cudaFuncSetAttribute(k_fwd_tc<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nt = ntiles(a), sms = sm_count();
    k_fwd_tc<D, W><<<nt < sms ? nt : sms, NTH, smem, s>>>(a, nt);
    return cudaGetLastError();
  }
  static cudaError_t bwd(const PassArgs& a, cudaStream_t s) {
    const size_t smem = bwd_smem();
    cudaError_t e = cudaFuncSetAttribute(k_bwd_tc<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nt = ntiles(a), sms = sm_count();
    const int64_t items = (int64_t)nt * a.N;
    k_bwd_tc<D, W><<<(int)(items < sms ? items : sms), NTH, smem, s>>>(a, nt, items);
    return cudaGetLastError();
  }
  static cudaError_t pack(const PassArgs& a, cudaStream_t s) {
    constexpr int per = Dm::Wp * (Dm::Dp / 8) + Dm::Wp * (Dm::Wp / 8) + Dm::Dp * (Dm::Wp / 8);
    const int64_t total = (int64_t)a.N * per;
    int grid = (int)((total + 255) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_pack_tc<D, W><<<grid, 256, 0, s>>>(a.params, static_cast<uint8_t*>(const_cast<void*>(a.wpack)), a.N);
    return cudaGetLastError();
  }
};

#define BSDE_TC_DIMS(X) X(100, 110) X(10, 20) X(37, 45)

}  // namespace tc

bool tc_supported(int d, int w) {
#define X(D_, W_) if (d == D_ && w == W_) return true;
  BSDE_TC_DIMS(X)
#undef X
  return false;
}

size_t tc_pack_bytes(int d, int w, int N, int) {
#define X(D_, W_) if (d == D_ && w == W_) return (size_t)N * tc::Dims<D_, W_>::WB;
  BSDE_TC_DIMS(X)
#undef X
  return 16;
}

size_t tc_xstore_bytes(int d, int w, int N, int64_t B_local) {
#define X(D_, W_) \
  if (d == D_ && w == W_) return (size_t)N * (size_t)((B_local + 127) / 128) * tc::Dims<D_, W_>::XB;
  BSDE_TC_DIMS(X)
#undef X
  return 16;
}


cudaError_t launch_fwd_tc(const PassArgs& a, cudaStream_t s) {
#define X(D_, W_) if (a.d == D_ && a.w == W_) return tc::Impl<D_, W_>::fwd(a, s);
  BSDE_TC_DIMS(X)
#undef X
  return cudaErrorNotSupported;
}
cudaError_t launch_bwd_tc(const PassArgs& a, cudaStream_t s) {
#define X(D_, W_) if (a.d == D_ && a.w == W_) return tc::Impl<D_, W_>::bwd(a, s);
  BSDE_TC_DIMS(X)
#undef X
  return cudaErrorNotSupported;
}
cudaError_t launch_pack_weights(const PassArgs& a, cudaStream_t s) {
#define X(D_, W_) if (a.d == D_ && a.w == W_) return tc::Impl<D_, W_>::pack(a, s);
  BSDE_TC_DIMS(X)
#undef X
  return cudaErrorNotSupported;
}

cudaError_t launch_umma_test(int mode, const float* A, const float* B, float* D, cudaStream_t s) {
  const size_t smem = 2 * (128 * 112 * 2 + 256) + 64;
  cudaError_t e = cudaFuncSetAttribute(tc::k_umma_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tc::k_umma_test<<<1, 128, smem, s>>>(mode, A, B, D);
  return cudaGetLastError();
}

cudaError_t launch_debug_dw_fast(uint32_t it, int n, int64_t m0, int64_t count, int d,
                                 float sqrt_dt, uint32_t k0, uint32_t k1, float* out,
                                 cudaStream_t s) {
  const int64_t th = count * ((d + 3) / 4);
  tc::k_debug_dw_fast<<<(int)((th + 255) / 256), 256, 0, s>>>(it, n, m0, count, d, sqrt_dt, k0, k1,
                                                             out);
  return cudaGetLastError();
}

}  // namespace bsde
