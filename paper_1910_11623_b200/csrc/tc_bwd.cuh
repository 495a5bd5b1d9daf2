// tc_bwd.cuh — adjoint pass on tcgen05.
//
// Step-major: each CTA owns a contiguous range of (n, tile) items, so it loads the
// step-n weight images ~once and keeps the three per-step weight-gradient
// accumulators (dW̃1 | dW̃2 | dW̃3, 3 × 112 fp32 columns) in TMEM across its range;
// they are flushed with fp32 atomics when the step changes.  Per item:
//   G1  A1 = X̃ W̃1ᵀ (recompute)        E1  H1 = ReLU(A1) (bf16 pairs, kept as the mask)
//   G2  A2 = H1 W̃2ᵀ                    E2  H2 = H1 + ReLU(A2) (bf16x2, as the forward)
//  [G3  Z = H2 W̃3ᵀ                     E3  HJB only: dZ needs Z]
//   G4  dH2 = dZ W̃3                    E4  dA2 = dH2 ⊙ 1[A2 > 0]
//   G5  dW̃3 += dZᵀ H2   (over the 128 paths of the tile, runs during E4)
//   G6  dH1 = dH2 + dA2 W̃2 (accumulated onto dH2 in TMEM)
//   G7  dW̃2 += dA2ᵀ H1  (runs during E6)
//                                       E6  dA1 = dH1 ⊙ 1[A1 > 0]
//   G8  dW̃1 += dA1ᵀ X̃   (issued behind the next item's G1, runs during its E1)
// with dZ = ā_{n+1}(ΔW_n - Δt ∂_z f) (R2; ΔW_n from the fp16
// path image written by the forward).  For the heat and Allen-Cahn drivers
// ∂_z f = 0, so dZ is formed from ΔW_n and ā alone, before G1, and the Z
// recompute is skipped.  The bias gradients come out of the constant-1 columns.
// No dX: X does not depend on θ.  ReLU'(0) = 0 (R15).
//
// The tensor pipe executes in issue order, so every chain GEMM (G1, G2, G4, G6)
// is issued before the gradient GEMM that can overlap the next epilogue; the
// commit after a chain GEMM also covers every earlier GEMM, which is what frees
// the operand buffers (H1 after G7, H2/dA2 after G5/G6/G7) without extra waits.
// The chain GEMMs G2, G4, G6 read their A operand (H1, dZ, dA2) from tensor
// memory, written by the epilogue next to the shared-memory copy the gradient
// GEMMs need: shared-memory bandwidth, which the SS MMAs nearly saturate, is the
// scarce resource of this kernel.
#pragma once

namespace bsde {
namespace tc {

template <int D, int W, bool NEEDZ>
__global__ void __launch_bounds__(NTH, 1) k_bwd_tc(PassArgs a, int ntiles, int64_t items) {
  using Dm = Dims<D, W>;
  constexpr int Dp = Dm::Dp, Wp = Dm::Wp;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* wimg = sm;
  uint8_t* const xb0 = sm + Dm::WB;
  uint8_t* const xb1 = sm + Dm::WB + Dm::ACT;
  auto xb = [&](int b) { return b ? xb1 : xb0; };
  uint8_t* hA = sm + Dm::WB + 2 * Dm::ACT;   // H1
  uint8_t* hB = hA + Dm::ACT;                // H2, then dA2
  uint8_t* hC = hB + Dm::ACT;                // dZ, then dA1
  // barriers: 0 weights, (1-2 unused), 3 chain GEMMs, 4 G8, 5 G5
  uint64_t* bars = reinterpret_cast<uint64_t*>(hC + Dm::ACT);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int q = warp & 3, g = warp >> 2;
  const int row = 32 * q + lane;
  // MMA / bulk-copy issuer: lane 0 of the highest warp, which the warp
  // schedulers favour (every GEMM of the chain waits on its issue)
  const bool issuer = t == NTH - 32;
  if (t == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = *tslot;
  const uint32_t lq = ((uint32_t)(32 * q) << 16) + 8u * g;
  // TMEM: chain accumulator | A operand of G2/G4/G6 (bf16 pairs) | dW̃1 | dW̃2 | dW̃3
  const uint32_t acc = tm, hT = tm + 112, GA1 = tm + 176, GA2 = tm + 288, GA3 = tm + 400;
  const uint32_t lrow = (uint32_t)(32 * q) << 16;

  const int64_t i0 = blockIdx.x * items / gridDim.x, i1 = (blockIdx.x + 1) * items / gridDim.x;
  const uint8_t* wsrc = static_cast<const uint8_t*>(a.wpack);
  const uint8_t* xst = static_cast<const uint8_t*>(a.xpack);
  const uint8_t* dst = static_cast<const uint8_t*>(a.dwpack);
  const NetDims nd{D, W};
  const float zc = -a.dt * driver_dfdz_coef(a.problem, a.lam);
  const float zc0 = -a.dt * driver_dfdz_const(a.problem);   // Black-Scholes: ∂_z f = r/σ
  const bool ac = per_step_abar(a.problem);
  constexpr uint32_t IW = idesc_bf16(128, Wp, false, false);     // G1, G2
  constexpr uint32_t ID = idesc_bf16(128, Dp, false, false);     // G3
  constexpr uint32_t IWm = idesc_bf16(128, Wp, false, true);     // G4, G6 (B = W̃ᵀ view)
  constexpr uint32_t IGW = idesc_bf16(128, Wp, true, true);      // G5, G7 (over paths)
  constexpr uint32_t IGD = idesc_bf16(128, Dp, true, true);      // G8

  // items are (step n, tile) in n-major order; (n, tile) is tracked incrementally
  // (a 64-bit division per item and thread costs more than an epilogue)
  auto img_of = [&](int n, int tile) -> size_t { return ((size_t)n * ntiles + tile) * Dm::XB; };
  // X̃ image of an item into its buffer: 16-byte cp.async by every thread (a bulk
  // copy would block its issuing thread for the copy's duration, ~800 cycles)
  auto load_x = [&](int64_t item, int n, int tile) {
    const int buf = (int)((item - i0) & 1);
    const uint8_t* src = xst + img_of(n, tile);
    uint8_t* dstp = xb(buf);
#pragma unroll
    for (int j = 0; j < (int)((Dm::XB / 16 + NTH - 1) / NTH); ++j) {
      const int c = t + j * NTH;
      if (c < (int)(Dm::XB / 16)) cp_async16(dstp + 16 * c, src + 16 * c);
    }
    cp_async_commit();
  };

  // per-path inputs of an item: ā_{n+1} and this thread's ΔW_n chunks (fp16)
  auto load_inputs = [&](int n, int tile, float& ab, float& pn, uint4 (&dwp)[4]) {
    const int64_t mloc = (int64_t)tile * 128 + row;
    // ā_{n+1} = ā_N P_N / P_{n+1}: both loaded here, divided where ā is used
    ab = mloc < a.B_local ? __ldg(a.abar + mloc) : 0.0f;
    pn = (ac && mloc < a.B_local) ? __ldcs(a.Pstore + (int64_t)n * a.B_local + mloc) : 1.0f;
    const uint8_t* src = dst + img_of(n, tile) + (row >> 3) * (Dp * 16) + (row & 7) * 16;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      dwp[i] = chunk_lt(g, i, Dp / 8) ? __ldcs(reinterpret_cast<const uint4*>(src + (g + 4 * i) * 128))
                                      : make_uint4(0, 0, 0, 0);
  };
  const int n_first = (int)(i0 / ntiles), t_first = (int)(i0 - (int64_t)n_first * ntiles);
  auto next_of = [&](int n, int tile, int& n1, int& t1) {
    t1 = tile + 1;
    n1 = n;
    if (t1 == ntiles) { t1 = 0; ++n1; }
  };
  int n_nx, t_nx;
  next_of(n_first, t_first, n_nx, t_nx);
  if (i0 < i1) load_x(i0, n_first, t_first);
  if (i0 + 1 < i1) load_x(i0 + 1, n_nx, t_nx);
  cp_async_wait_all();
  fence_async_smem();
  __syncthreads();
  float ab = 0.0f, pn = 1.0f;
  uint4 dwp[4];
  if (i0 < i1) load_inputs(n_first, t_first, ab, pn, dwp);

  uint32_t mph = 0, wph = 0, g8ph = 0, g5ph = 0;
  unsigned long long* const clk = (a.clk && blockIdx.x == 0 && t == 32) ? a.clk : nullptr;
#define CLK(i) do { if (item - i0 < 64) BSDE_STAMP(clk, (item - i0) * 16 + (i)); } while (0)
  int cur_n = -1;
  bool f5 = false, f7 = false, f8 = false;   // accumulator holds a partial of step cur_n
  bool g8_pending = false;                   // G8 of the previous item not issued yet

  // G8 of the previous item (dA1 in hC, its X̃ in xb(pbuf)); thread 0
  auto issue_g8 = [&](int pbuf) {
    gemm(GA1, mnmaj(hC, Wp), mnmaj(xb(pbuf), Dp), 128 / 16, IGD, f8);
    mma_commit(&bars[4]);
  };
  // gradient flush of step cur_n: TMEM -> fp32 atomics (lane = gradient row)
  auto flush = [&](int pbuf) {
    if (issuer) {
      tc_after();
      if (g8_pending) issue_g8(pbuf);
      else mma_commit(&bars[4]);   // covers every GEMM issued so far
    }
    g8_pending = false;
    mbar_wait(&bars[4], g8ph);
    g8ph ^= 1;
    tc_after();
    // deterministic mode: this CTA's partial of step cur_n, every entry stored once
    float* G = a.dpart ? a.dpart + ((int64_t)blockIdx.x * a.dseg + (cur_n - (int)(i0 / ntiles))) *
                                      nd.step_size()
                       : a.grad + nd.step_base(cur_n);
    const bool det = a.dpart != nullptr;
    auto put = [&](float* p, float x) { if (det) *p = x; else atomicAdd(p, x); };
    float v[32];
    tmem_ld_g4(GA1 + lq, g, Dp / 8, v);               // dW̃1 row = w-unit, cols = d-inputs
    if (row < W) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int k = 8 * (g + 4 * (i / 8)) + (i % 8);
        if (k < D) put(G + nd.off_W1() + row * D + k, v[i]);
        else if (k == D) put(G + nd.off_b1() + row, v[i]);
      }
    }
    tmem_ld_g4(GA2 + lq, g, Wp / 8, v);               // dW̃2
    if (row < W) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int k = 8 * (g + 4 * (i / 8)) + (i % 8);
        if (k < W) put(G + nd.off_W2() + row * W + k, v[i]);
        else if (k == W) put(G + nd.off_b2() + row, v[i]);
      }
    }
    tmem_ld_g4(GA3 + lq, g, Wp / 8, v);               // dW̃3 row = d-output
    if (row < D) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int k = 8 * (g + 4 * (i / 8)) + (i % 8);
        if (k < W) put(G + nd.off_W3() + row * W + k, v[i]);
        else if (k == W) put(G + nd.off_b3() + row, v[i]);
      }
    }
    tc_before();
    __syncthreads();
  };

  int n = n_first, tile = t_first;
  for (int64_t item = i0; item < i1; ++item, n = n_nx, tile = t_nx) {
    next_of(n, tile, n_nx, t_nx);
    const int k = (int)(item - i0), buf = k & 1;
    if (n != cur_n) {
      if (cur_n >= 0) flush(buf ^ 1);
      if (issuer) {   // the weight images' last readers completed in flush
        mbar_expect_tx(&bars[0], Dm::WB);
        const uint8_t* src = wsrc + (size_t)n * Dm::WB;
        for (uint32_t off = 0; off < Dm::WB; off += 16384u)
          bulk_g2s(wimg + off, src + off, min(16384u, Dm::WB - off), &bars[0]);
      }
      mbar_wait(&bars[0], wph);
      wph ^= 1;
      cur_n = n;
      f5 = f7 = f8 = false;
    }
    CLK(0);
    const bool g8_now = g8_pending;
    if (issuer) {   // G1 (recompute), then the previous item's G8
      tc_after();
      gemm(acc, kmaj(xb(buf), Dp), kmaj(wimg, Dp), Dp / 16, IW, false);
      mma_commit(&bars[3]);
      if (g8_now) issue_g8(buf ^ 1);
    }
    if (g8_now) f8 = true;
    g8_pending = false;
    // dZ of this item (heat, Allen-Cahn: ∂_z f = 0; Black-Scholes: the constant r/σ), bf16 pairs: stored into hC
    // (G5) once G8 of the previous item has read dA1 from it, and into hT (G4)
    // once G2 has read H1 from it
    uint4 dzp[4];
    const float ab_i = ac ? __fdividef(ab, pn) : ab;
    const float abz0 = ab_i * zc0;   // ā(ΔW - Δt ∂_z f) with the constant part of ∂_z f
    uint4 dwc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) dwc[i] = dwp[i];
    if (!NEEDZ) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float dw[8];
        unpack_dw(dwc[i], dw);
#pragma unroll
        for (int e = 0; e < 8; ++e) dw[e] = col_lt(g, i, e, D) ? fmaf(ab_i, dw[e], abz0) : 0.0f;
        dzp[i] = make_uint4(pack2(dw[0], dw[1]), pack2(dw[2], dw[3]), pack2(dw[4], dw[5]),
                            pack2(dw[6], dw[7]));
      }
    }
    if (item + 1 < i1) load_inputs(n_nx, t_nx, ab, pn, dwp);   // consumed by the next item
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(1);
    tc_after();
    // H1 = ReLU(A1) and R2 = ReLU(A2) as bf16 pairs: operands, and (non-zero) the
    // ReLU masks 1[A1 > 0], 1[A2 > 0] of E6 / E4
    uint4 h1p[4], r2p[4];
    {  // E1: H1 -> hA (G7; its last reader, G7 of the previous item, is done) and hT (G2)
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        h1p[i] = make_uint4(relu_pack2(v[8 * i], v[8 * i + 1]), relu_pack2(v[8 * i + 2], v[8 * i + 3]),
                            relu_pack2(v[8 * i + 4], v[8 * i + 5]), relu_pack2(v[8 * i + 6], v[8 * i + 7]));
        if (chunk_lt(g, i, Wp / 8)) {
          tmem_st4(hT + lrow + 4u * (g + 4 * i), h1p[i]);
          st_chunk_u4(hA, row, g + 4 * i, Wp, h1p[i]);
        }
      }
    }
    // No proxy fence here: G2 reads H1 from TMEM; the smem copy (G7's operand) is
    // fenced with dA2 later.  fence.proxy.async is a MEMBAR.ALL.CTA, which would
    // also wait for this item's prefetch loads from HBM.
    tmem_wait_st();
    tc_before();
    __syncthreads();
    CLK(2);
    if (issuer) {   // G2: A2 = H1 W̃2ᵀ (A in TMEM)
      tc_after();
      gemm_ta(acc, hT, kmaj(wimg + Dm::W1B, Wp), Wp / 16, IW, false);
      mma_commit(&bars[3]);
    }
    if (g8_now) {   // G8 (previous item) has read hC and its X̃ buffer
      mbar_wait(&bars[4], g8ph);
      g8ph ^= 1;
    }
    if (k > 0 && item + 1 < i1) load_x(item + 1, n_nx, t_nx);
    if (!NEEDZ) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Dp / 8)) st_chunk_u4(hC, row, g + 4 * i, Dp, dzp[i]);
    }
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(3);
    tc_after();
    {  // E2: H2 = H1 + ReLU(A2) in bf16x2 arithmetic (R17, as in the forward) -> hB (G5)
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        r2p[i] = make_uint4(relu_pack2(v[8 * i], v[8 * i + 1]), relu_pack2(v[8 * i + 2], v[8 * i + 3]),
                            relu_pack2(v[8 * i + 4], v[8 * i + 5]), relu_pack2(v[8 * i + 6], v[8 * i + 7]));
        if (chunk_lt(g, i, Wp / 8))
          st_chunk_u4(hB, row, g + 4 * i, Wp,
                      make_uint4(bf2_add(h1p[i].x, r2p[i].x), bf2_add(h1p[i].y, r2p[i].y),
                                 bf2_add(h1p[i].z, r2p[i].z), bf2_add(h1p[i].w, r2p[i].w)));
      }
      if (!NEEDZ) {   // dZ -> hT (G2 has read H1)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (chunk_lt(g, i, Dp / 8)) tmem_st4(hT + lrow + 4u * (g + 4 * i), dzp[i]);
      }
    }
    tmem_wait_st();
    fence_async_smem();
    tc_before();
    __syncthreads();
    CLK(4);
    if (NEEDZ) {   // G3: Z = H2 W̃3ᵀ; E3: dZ = ā(ΔW - Δt ∂_z f) -> hC, hT
      if (issuer) {
        tc_after();
        gemm(acc, kmaj(hB, Wp), kmaj(wimg + Dm::W1B + Dm::W2B, Wp), Wp / 16, ID, false);
        mma_commit(&bars[3]);
      }
      mbar_wait(&bars[3], mph);
      mph ^= 1;
      tc_after();
      float z[32];
      tmem_ld4x8(acc + lq, z);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float dw[8];
        unpack_dw(dwc[i], dw);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          z[8 * i + e] = col_lt(g, i, e, D) ? fmaf(ab_i, fmaf(zc, z[8 * i + e], dw[e]), abz0) : 0.0f;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Dp / 8)) {
          const uint4 u = make_uint4(pack2(z[8 * i], z[8 * i + 1]), pack2(z[8 * i + 2], z[8 * i + 3]),
                                     pack2(z[8 * i + 4], z[8 * i + 5]), pack2(z[8 * i + 6], z[8 * i + 7]));
          st_chunk_u4(hC, row, g + 4 * i, Dp, u);
          tmem_st4(hT + lrow + 4u * (g + 4 * i), u);
        }
      tmem_wait_st();
      fence_async_smem();
      tc_before();
      __syncthreads();
    }
    CLK(5);
    if (issuer) {
      tc_after();
      // G4: dH2 = dZ W̃3 (A in TMEM) ; G5: dW̃3 += dZᵀ H2
      gemm_ta(acc, hT, mnmaj(wimg + Dm::W1B + Dm::W2B, Wp), Dp / 16, IWm, false);
      mma_commit(&bars[3]);
      gemm(GA3, mnmaj(hC, Dp), mnmaj(hB, Wp), 128 / 16, IGW, f5);
      mma_commit(&bars[5]);
    }
    f5 = true;
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(6);
    tc_after();
    uint4 pk[4];
    {  // E4: dA2 = dH2 ⊙ 1[A2 > 0] -> hT (G6), later over H2 in hB (G7)
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        pk[i] = make_uint4(pack2(v[8 * i], v[8 * i + 1]) & nz_mask2(r2p[i].x),
                           pack2(v[8 * i + 2], v[8 * i + 3]) & nz_mask2(r2p[i].y),
                           pack2(v[8 * i + 4], v[8 * i + 5]) & nz_mask2(r2p[i].z),
                           pack2(v[8 * i + 6], v[8 * i + 7]) & nz_mask2(r2p[i].w));
        if (chunk_lt(g, i, Wp / 8)) tmem_st4(hT + lrow + 4u * (g + 4 * i), pk[i]);
      }
    }
    tmem_wait_st();
    tc_before();
    __syncthreads();
    CLK(7);
    if (issuer) {   // G6: dH1 = dH2 + dA2 W̃2 (accumulated onto dH2; A in TMEM)
      tc_after();
      gemm_ta(acc, hT, mnmaj(wimg + Dm::W1B, Wp), Wp / 16, IWm, true);
      mma_commit(&bars[3]);
    }
    // dA2 over H2 once G5 has read it, then G7: dW̃2 += dA2ᵀ H1 (runs during E6)
    mbar_wait(&bars[5], g5ph);
    g5ph ^= 1;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (chunk_lt(g, i, Wp / 8)) st_chunk_u4(hB, row, g + 4 * i, Wp, pk[i]);
    fence_async_smem();
    __syncthreads();
    CLK(8);
    if (issuer) {
      tc_after();
      gemm(GA2, mnmaj(hB, Wp), mnmaj(hA, Wp), 128 / 16, IGW, f7);
    }
    f7 = true;
    mbar_wait(&bars[3], mph);
    mph ^= 1;
    CLK(9);
    tc_after();
    {  // E6: dA1 = dH1 ⊙ 1[A1 > 0] -> hC (dZ's readers G4, G5 are done)
      float v[32];
      tmem_ld4x8(acc + lq, v);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (chunk_lt(g, i, Wp / 8))
          st_chunk_u4(hC, row, g + 4 * i, Wp,
                      make_uint4(pack2(v[8 * i], v[8 * i + 1]) & nz_mask2(h1p[i].x),
                                 pack2(v[8 * i + 2], v[8 * i + 3]) & nz_mask2(h1p[i].y),
                                 pack2(v[8 * i + 4], v[8 * i + 5]) & nz_mask2(h1p[i].z),
                                 pack2(v[8 * i + 6], v[8 * i + 7]) & nz_mask2(h1p[i].w)));
    }
    cp_async_wait_all();   // the next item's X̃ (loaded during this item) is in place
    fence_async_smem();
    tc_before();
    __syncthreads();
    g8_pending = true;
    CLK(10);
  }
  if (cur_n >= 0) flush((int)((i1 - i0 - 1) & 1));
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 512);
  }
#undef CLK
}

}  // namespace tc
}  // namespace bsde
