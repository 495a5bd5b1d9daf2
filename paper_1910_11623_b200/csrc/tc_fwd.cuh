// tc_fwd.cuh — forward rollout on tcgen05:
// one 128-path tile (4 threads per path, TMEM lane = path) walks all N steps.
// Per step: the X_n operand image (written by k_paths_tc) is bulk-copied into
// shared memory, the three GEMMs A1 = X̃ W̃1ᵀ, A2 = H1 W̃2ᵀ, Z = H2 W̃3ᵀ run on the
// tensor cores with fp32 accumulators in TMEM (weights double-buffered), the
// epilogues form H1 = ReLU(A1), H2 = H1 + ReLU(A2) (Eq. 7, h = 1) and the Y
// update Y_{n+1} = Y_n - f(Y_n, Z_n) Δt + Z_n·ΔW_n (Eq. 5, φ = -f, R2).  The
// terminal residual R = Y_N - g(X_N) (Eq. 6) uses |X_N|² from k_paths_tc.
#pragma once

namespace bsde {
namespace tc {

template <int D, int W>
__global__ void __launch_bounds__(NTH, 1) k_fwd_tc(PassArgs a, int ntiles) {
  using Dm = Dims<D, W>;
  constexpr int Dp = Dm::Dp, Wp = Dm::Wp;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* wimg0 = sm;
  uint8_t* wimg1 = sm + Dm::WB;
  uint8_t* xop = sm + 2 * Dm::WB;
  uint8_t* hop = xop + Dm::ACT;
  float2* red = reinterpret_cast<float2*>(hop + Dm::ACT);            // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 4 * 128);       // 0,1 weights, 2 mma, 3 X
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  __shared__ double lred[4];
  __shared__ float gred[4];

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int q = warp & 3, g = warp >> 2;
  const int row = 32 * q + lane;
  if (t == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
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
  const uint8_t* xst = static_cast<const uint8_t*>(a.xpack);
  const uint8_t* dst = static_cast<const uint8_t*>(a.dwpack);
  const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int64_t total_seq = (int64_t)my_tiles * N;
  constexpr uint32_t I1 = idesc_bf16(128, Wp, false, false);
  constexpr uint32_t I3 = idesc_bf16(128, Dp, false, false);

  // sequence s = (k-th tile of this CTA) * N + n
  auto img_of = [&](int64_t s) -> size_t {
    const int tile = (int)blockIdx.x + (int)(s / N) * (int)gridDim.x;
    return ((size_t)(s % N) * ntiles + tile) * Dm::XB;
  };
  auto load_weights = [&](int64_t s) {   // thread 0
    const int n = (int)(s % N);
    uint8_t* dstw = (s & 1) ? wimg1 : wimg0;
    uint64_t* bar = &bars[s & 1];
    mbar_expect_tx(bar, Dm::WB);
    const uint8_t* src = wsrc + (size_t)n * Dm::WB;
    for (uint32_t off = 0; off < Dm::WB; off += 16384u)
      bulk_g2s(dstw + off, src + off, min(16384u, Dm::WB - off), bar);
  };
  auto load_x = [&](int64_t s) {         // thread 0: X_n operand image into xop
    mbar_expect_tx(&bars[3], Dm::XB);
    bulk_g2s(xop, xst + img_of(s), Dm::XB, &bars[3]);
    if (s + 2 < total_seq) bulk_prefetch_l2(xst + img_of(s + 2), Dm::XB);
  };
  if (t == 0 && total_seq > 0) {
    load_weights(0);
    load_x(0);
    if (total_seq > 1) bulk_prefetch_l2(xst + img_of(1), Dm::XB);
  }

  unsigned long long* const clk = (a.clk && blockIdx.x == 0 && t == 32) ? a.clk : nullptr;
#define CLK(i) do { if (clk && s < 64) clk[s * 16 + (i)] = clock64(); } while (0)
  uint32_t mph = 0;
  int64_t s = 0;
  double lsum = 0.0;
  float dy0 = 0.0f;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t mloc = (int64_t)tile * 128 + row;
    const bool valid = mloc < a.B_local;
    float Y = a.params[0];
    for (int n = 0; n < N; ++n, ++s) {
      CLK(0);
      uint8_t* wimg = (s & 1) ? wimg1 : wimg0;
      if (t == 0) {
        if (s + 1 < total_seq) load_weights(s + 1);
        mbar_wait(&bars[3], (uint32_t)(s & 1));            // X_n image
        mbar_wait(&bars[s & 1], (uint32_t)((s >> 1) & 1)); // weights of step n
        tc_after();
        gemm(tm, kmaj(xop, Dp), kmaj(wimg, Dp), Dp / 16, I1, false);                  // A1
        mma_commit(&bars[2]);
      }
      uint4 dwp[4];                                   // ΔW_n chunks (fp16), needed at epi3
      {
        const uint8_t* src = dst + img_of(s) + (row >> 3) * (Dp * 16) + (row & 7) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dwp[i] = chunk_lt(g, i, Dp / 8) ? __ldcs(reinterpret_cast<const uint4*>(src + (g + 4 * i) * 128))
                                          : make_uint4(0, 0, 0, 0);
      }
      mbar_wait(&bars[2], mph);
      mph ^= 1;
      CLK(1);
      if (t == 0 && s + 1 < total_seq) load_x(s + 1);   // G1 has consumed xop
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
      __syncthreads();
      CLK(2);
      if (t == 0) {
        tc_after();
        gemm(tm + 128, kmaj(hop, Wp), kmaj(wimg + Dm::W1B, Wp), Wp / 16, I1, false);   // A2
        mma_commit(&bars[2]);
      }
      if (n > 0) {   // finish a4 of step n-1 from the partial sums of the four threads
        const float2 r0 = red[row], r1 = red[128 + row], r2 = red[256 + row], r3 = red[384 + row];
        const float cz = (r0.x + r1.x) + (r2.x + r3.x), zz = (r0.y + r1.y) + (r2.y + r3.y);
        Y = Y - driver_f(a.problem, Y, zz, a.lam) * a.dt + cz;
      }
      if (!a.eval && a.problem == kAllenCahn && valid && g == 0)
        a.Ystore[(int64_t)n * a.B_local + mloc] = Y;
      mbar_wait(&bars[2], mph);
      mph ^= 1;
      CLK(3);
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
      __syncthreads();
      CLK(4);
      if (t == 0) {
        tc_after();
        gemm(tm, kmaj(hop, Wp), kmaj(wimg + Dm::W1B + Dm::W2B, Wp), Wp / 16, I3, false);  // Z
        mma_commit(&bars[2]);
      }
      mbar_wait(&bars[2], mph);
      mph ^= 1;
      CLK(5);
      tc_after();
      float cz = 0.0f, zz = 0.0f;
      {  // a4 partials c = Z·ΔW, |Z|²
        float z[32];
        tmem_ld4x8(acc0, z);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float dw[8];
          unpack_dw(dwp[i], dw);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if (col_lt(g, i, e, D)) {
              cz = fmaf(z[8 * i + e], dw[e], cz);
              zz = fmaf(z[8 * i + e], z[8 * i + e], zz);
            }
          }
        }
      }
      red[g * 128 + row] = make_float2(cz, zz);   // a4 is finished after the next barrier
      tc_before();
      CLK(6);
    }
    __syncthreads();
    {
      const float2 r0 = red[row], r1 = red[128 + row], r2 = red[256 + row], r3 = red[384 + row];
      const float cz = (r0.x + r1.x) + (r2.x + r3.x), zz = (r0.y + r1.y) + (r2.y + r3.y);
      Y = Y - driver_f(a.problem, Y, zz, a.lam) * a.dt + cz;                         // a4, n = N-1
    }
    __syncthreads();   // red is rewritten by the next tile
    // a5: R = Y_N - g(X_N); loss; ā recursion and dY0
    if (g == 0 && valid) {
      const float R = Y - terminal_g(a.problem, a.xn2[mloc]);
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
  }
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, 256);
  }
#undef CLK
}

}  // namespace tc
}  // namespace bsde
