// tc_bwd.cuh — adjoint pass on tcgen05.
//
// Step-major: each CTA owns a contiguous range of (n, tile) items, so it loads the
// step-n weight images ~once and keeps the three per-step weight-gradient
// accumulators (dW̃1 | dW̃2 | dW̃3, 3 × 112 fp32 columns) in TMEM across its range;
// they are flushed with fp32 atomics when the step changes.  Per item: recompute
// A1, A2, Z from the X_n image (bulk-copied, double-buffered), form
// dZ = ā_{n+1}(ΔW_n - Δt ∂_z f) (ΔW_n from the fp16 path image), then
//   G4 dH2 = dZ W̃3            G5 dW̃3 += dZᵀ H2     (contraction over the 128 paths)
//   G6 dH1 = dH2 + dA2 W̃2     G7 dW̃2 += dA2ᵀ H1
//                              G8 dW̃1 += dA1ᵀ X̃
// with dA2 = dH2 ⊙ 1[A2 > 0], dA1 = dH1 ⊙ 1[A1 > 0] (R15); the bias gradients come
// out of the constant-1 columns.  No dX: X does not depend on θ.
#pragma once

namespace bsde {
namespace tc {

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
  const uint8_t* dst = static_cast<const uint8_t*>(a.dwpack);
  const NetDims nd{D, W};
  const float zc = -a.dt * driver_dfdz_coef(a.problem, a.lam);
  constexpr uint32_t IW = idesc_bf16(128, Wp, false, false);     // G1, G2
  constexpr uint32_t ID = idesc_bf16(128, Dp, false, false);     // G3
  constexpr uint32_t IWm = idesc_bf16(128, Wp, false, true);     // G4, G6 (B = W̃ᵀ view)
  constexpr uint32_t IGW = idesc_bf16(128, Wp, true, true);      // G5, G7 (over paths)
  constexpr uint32_t IGD = idesc_bf16(128, Dp, true, true);      // G8

  auto img_of = [&](int64_t item) -> size_t {
    const int n = (int)(item / ntiles), tile = (int)(item - (int64_t)n * ntiles);
    return ((size_t)n * ntiles + tile) * Dm::XB;
  };
  auto load_x = [&](int64_t item) {   // thread 0
    const int buf = (int)((item - i0) & 1);
    uint64_t* bar = &bars[1 + buf];
    mbar_expect_tx(bar, Dm::XB);
    bulk_g2s(buf ? xbuf1 : xbuf0, xst + img_of(item), Dm::XB, bar);
    if (item + 2 < i1) bulk_prefetch_l2(xst + img_of(item + 2), Dm::XB);
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
    const float ab = valid ? (a.problem == kAllenCahn ? a.abar[(int64_t)n * a.B_local + mloc]
                                                      : a.abar[mloc])
                           : 0.0f;
    if (t == 0) {   // G1: A1 = X̃ W̃1ᵀ (recompute)
      mbar_wait(&bars[1 + buf], (uint32_t)(((item - i0) >> 1) & 1));
      tc_after();
      gemm(acc, kmaj(xop, Dp), kmaj(wimg, Dp), Dp / 16, IW, false);
      mma_commit(&bars[3]);
    }
    uint4 dwp[4];   // ΔW_n (fp16 path image), needed at the dZ epilogue
    {
      const uint8_t* src = dst + img_of(item) + (row >> 3) * (Dp * 16) + (row & 7) * 16;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dwp[i] = chunk_lt(g, i, Dp / 8) ? __ldcs(reinterpret_cast<const uint4*>(src + (g + 4 * i) * 128))
                                        : make_uint4(0, 0, 0, 0);
    }
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
        if (chunk_lt(g, i, Wp / 8)) st_chunk(hop, row, g + 4 * i, Wp, v + 8 * i);
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
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(5);
    tc_after();
    {  // dZ = ā_{n+1}(ΔW_n - Δt ∂_z f), columns >= D zero
      float z[32];
      tmem_ld4x8(acc + lq, z);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float dw[8];
        unpack_dw(dwp[i], dw);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          z[8 * i + e] = col_lt(g, i, e, D) ? ab * fmaf(zc, z[8 * i + e], dw[e]) : 0.0f;
      }
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
        if (chunk_lt(g, i, Wp / 8)) st_chunk(b2, row, g + 4 * i, Wp, v + 8 * i);
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
        if (chunk_lt(g, i, Wp / 8)) st_chunk(b3, row, g + 4 * i, Wp, v + 8 * i);
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

}  // namespace tc
}  // namespace bsde
