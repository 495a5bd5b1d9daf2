// tc_fwd.cuh — forward rollout on tcgen05, one fused
// pass; CTAs are persistent over 128-path tiles, every tile walks all N steps.
//
// Work split (12 worker warps + 1 control warp, 416 threads; 13 warps keep the
// 128-register budget that 17 would cut to 96):
//  * worker warp w serves TMEM lane quadrant q = w % 4 (paths 32q..32q+31 of the
//    tile, one path per lane) and column group g = w / 4: the 8-column chunks
//    c = g, g+3, g+6, ... of every 112-column image.  Every worker both draws
//    its share of the Brownian increments ΔW_n = √Δt·z (Philox4x32-10 +
//    Box-Muller, R8) and runs its share of the network epilogues;
//    the Euler state X_{n+1} = X_n + √2 ΔW_n (Eq. 5) of its columns
//    stays in exact fp32 registers, ΔW_n in binary16 registers until the Y
//    update reads it.
//  * the control warp issues the tcgen05 MMAs (lane 0) once all workers have
//    arrived at the named barrier of the stage, and streams the per-step weight
//    images into shared memory with bulk copies.  Workers never wait at a
//    barrier: they arrive and continue with the next slice of random numbers,
//    and wait only for the completion of the MMA whose result they read.
//
// One step n of a tile (Eq. 7, h = 1; R4):
//    workers: X̃_n (bf16 operand, constant-1 column folds b1) -> TMEM  | arrive B_X
//    control: G1  A1 = X̃_n W̃1ᵀ                        (A from TMEM)
//    workers: slice 1 of ΔW_n   | wait G1 | E1 H1 = ReLU(A1) -> TMEM    | arrive B_1
//    control: G2  A2 = H1 W̃2ᵀ                         (A from TMEM)
//    workers: slice 2 of ΔW_n   | wait G2 | E2 H2 = H1 + ReLU(A2)       | arrive B_2
//    control: G3  Z = H2 W̃3ᵀ                          (A from TMEM)
//    workers: slice 3           | wait G3 | E3 partial sums of Z·ΔW (|Z|², Σ Z)
//             over the worker's columns | X̃_{n+1} -> TMEM             | arrive B_X
// A slice is three of the worker's Philox blocks (12 increments), each folded
// into X at once; ~500 cycles of the SM's issue, longer than the GEMM it hides
// (~420), so the tensor pipe and the epilogues stay off the critical path.
// The Y update Y_{n+1} = Y_n - f(Y_n, Z_n)Δt + Z_n·ΔW_n (Eq. 5, R2) of path m is
// finished by its group-0 worker from the three partial sums during E1 of the
// next step (the partials are complete once G1 of the next step has been
// issued, which waits for every worker).  The terminal residual
// R = Y_N - g(X_N) (Eq. 6) and the scalar adjoint ā close each tile.  The
// X̃_n (bf16) and ΔW_n (fp16) images go to global memory for the adjoint
// (DESIGN.md §5).
#pragma once

namespace bsde {
namespace tc {

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// ΔW chunk from its fp16 image (16 bytes -> 8 floats)
__device__ __forceinline__ void unpack_dw(const uint4& u, float* v) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}

constexpr int kFwdGroups = 3;                                   // column groups per path
constexpr int kFwdWorkers = 128 * kFwdGroups, kFwdWorkerWarps = kFwdWorkers / 32;
constexpr int kFwdThreads = kFwdWorkers + 32;
// named barriers: X̃_n written (before G1), E1 done (before G2), E2 done (before
// G3), workers only (tile tail)
constexpr int kBarX = 1, kBarE1 = 2, kBarE2 = 3, kBarTail = 4;

// Predicates on a worker's column chunk c = g + 3i (g = 0, 1, 2 the column group,
// warp-uniform) that fold at compile time once i and the offset are constants
// (after unrolling): true for every g when the largest c satisfies them, false
// for every g when the smallest does not; only the rest is a runtime test.
__device__ __forceinline__ bool chunk_lt3(int g, int i, int LIM) {
  return (kFwdGroups - 1 + kFwdGroups * i < LIM) || (kFwdGroups * i < LIM && g + kFwdGroups * i < LIM);
}
// column 8c + off < LIM
__device__ __forceinline__ bool col_lt3(int g, int i, int off, int LIM) {
  return (8 * (kFwdGroups - 1 + kFwdGroups * i) + off < LIM) ||
         (8 * kFwdGroups * i + off < LIM && 8 * (g + kFwdGroups * i) + off < LIM);
}

// Block b of a worker (columns 8c + 4(b%2), c = g + 3(b/2)) lies below D for every
// column group / for none: compile-time facts that split a slice into an
// unconditional prefix and single blocks behind a warp-uniform branch.
__host__ __device__ constexpr bool blk_all(int b, int D) {
  return 8 * (kFwdGroups - 1 + kFwdGroups * (b / 2)) + 4 * (b % 2) < D;
}
__host__ __device__ constexpr bool blk_none(int b, int D) {
  return 8 * kFwdGroups * (b / 2) + 4 * (b % 2) >= D;
}
__host__ __device__ constexpr int blk_prefix(int b0, int b1, int D) {   // first not-all-valid block
  return b0 >= b1 ? b1 : (blk_all(b0, D) ? blk_prefix(b0 + 1, b1, D) : b0);
}

// Rounds 0-2 of Philox4x32-10 on the counter (q, m, n, it) (R8): every product except
// the two that involve the path index m depends on (q, n, it, key) only, so they are
// computed once per launch for every (step n, block q) into shared memory, and a lane
// starts each block at round 1's m-dependent multiply (16 IMAD.WIDE instead of 20).
// Row entry (A, B, C, D) and E, with (round 0) lo0 = M0 q, hi0 = hi(M0 q), lo1 = M1 n,
// hi1 = hi(M1 n), z1 = hi0 ^ it ^ k1; (round 1) x2 = hi(M1 z1) ^ lo1 ^ (k0 + W0),
// y2 = M1 z1:
//   A = hi1 ^ k0              x1 = A ^ m
//   B = lo0 ^ (k1 + W1)       z2 = hi(M0 x1) ^ B,   w2 = M0 x1
//   C = y2 ^ (k0 + 2 W0)      x3 = hi(M1 z2) ^ C,   y3 = M1 z2
//   D = hi(M0 x2) ^ (k1 + 2 W1)   z3 = D ^ w2
//   E = M0 x2                 w3 = E
__device__ __forceinline__ void fwd_philox_table(uint4* tab4, uint32_t* tabE, int nq, int nsteps, uint32_t it,
                                                 uint32_t k0, uint32_t k1) {
  for (int i = threadIdx.x; i < nq * nsteps; i += blockDim.x) {
    const uint32_t q = (uint32_t)(i % nq), n = (uint32_t)(i / nq);
    const uint32_t lo0 = kPhiloxM0 * q, hi0 = __umulhi(kPhiloxM0, q);
    const uint32_t lo1 = kPhiloxM1 * n, hi1 = __umulhi(kPhiloxM1, n);
    const uint32_t z1 = hi0 ^ it ^ k1;
    const uint32_t x2 = __umulhi(kPhiloxM1, z1) ^ lo1 ^ (k0 + kPhiloxW0), y2 = kPhiloxM1 * z1;
    tab4[i] = make_uint4(hi1 ^ k0, lo0 ^ (k1 + kPhiloxW1), y2 ^ (k0 + 2u * kPhiloxW0),
                         __umulhi(kPhiloxM0, x2) ^ (k1 + 2u * kPhiloxW1));
    tabE[i] = kPhiloxM0 * x2;
  }
}

// Increments of the worker's Philox blocks b = B0 .. B0+NB-1 of step n: block b
// holds columns 8c + 4(b%2) .. +3 of chunk c = g + 3(b/2), i.e. counter word 0
// q = 2c + b%2 (R8).  Interleaved for ILP; blocks whose columns are all >= D
// are skipped (the test is warp-uniform: g depends on the warp only) and read
// as 0.  Coupled paths (cpl > 1, NEXT-3): the sum over the cpl fine steps
// n·cpl + j of √(Δt/cpl)·z (sdt = √(Δt/cpl)); the uncoupled instance (CPL false)
// keeps the loop out of the hot code.
template <int D, int B0, int NB, bool CPL, bool TAB>
__device__ __forceinline__ void gen_blocks(int g, uint32_t m, uint32_t n, uint32_t it, uint32_t k0,
                                           uint32_t k1, float sdt, float (&z)[4 * NB], int cpl,
                                           const uint4* tab4, const uint32_t* tabE) {
  auto one = [&](uint32_t nf, bool add) {   // the normals of (fine) step nf
    uint4 c[NB];
    bool ok[NB];
    constexpr int NQ = Dims<D, 8>::Dp / 4;   // Philox blocks per path-step (table row)
    constexpr bool tab = !CPL && TAB;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int b = B0 + j, q = 2 * (g + kFwdGroups * (b / 2)) + b % 2;
      ok[j] = col_lt3(g, b / 2, 4 * (b % 2), D);   // 4q < D
      if (tab) {   // rounds 0-2 from the step's table row (fwd_philox_table); only the
                   // two multiplies that involve the path index m remain per lane
        const uint4 u = tab4[nf * NQ + q];
        const uint32_t x1 = u.x ^ m;
        const uint32_t l0 = kPhiloxM0 * x1, h0 = __umulhi(kPhiloxM0, x1);
        const uint32_t z2 = h0 ^ u.y;
        const uint32_t m1 = kPhiloxM1 * z2, g1 = __umulhi(kPhiloxM1, z2);
        c[j] = make_uint4(g1 ^ u.z, m1, u.w ^ l0, tabE[nf * NQ + q]);
      } else {
        c[j] = make_uint4((uint32_t)q, m, nf, it);
      }
    }
    constexpr int r0 = tab ? 3 : 0;
    uint32_t a0 = k0 + (uint32_t)r0 * kPhiloxW0, a1 = k1 + (uint32_t)r0 * kPhiloxW1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r < r0) continue;
      if (r > r0) { a0 += kPhiloxW0; a1 += kPhiloxW1; }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (!ok[j]) continue;
        const uint32_t lo0 = kPhiloxM0 * c[j].x, hi0 = __umulhi(kPhiloxM0, c[j].x);
        const uint32_t lo1 = kPhiloxM1 * c[j].z, hi1 = __umulhi(kPhiloxM1, c[j].z);
        c[j] = make_uint4(hi1 ^ c[j].y ^ a0, lo1, hi0 ^ c[j].w ^ a1, lo0);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (ok[j]) {
        box_muller_fast(c[j].x, c[j].y, sdt, v[0], v[1]);
        box_muller_fast(c[j].z, c[j].w, sdt, v[2], v[3]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) z[4 * j + e] = add ? z[4 * j + e] + v[e] : v[e];
    }
  };
  if constexpr (!CPL) {
    one(n, false);
  } else {
    one(n * (uint32_t)cpl, false);
#pragma unroll 1
    for (int jf = 1; jf < cpl; ++jf) one(n * (uint32_t)cpl + (uint32_t)jf, true);
  }
}

template <int D, int W>
struct FwdSmem {
  using Dm = Dims<D, W>;
  static constexpr uint32_t W1 = 0, W2 = Dm::W1B, W3 = Dm::W1B + Dm::W2B;   // weight images
  // partial sums per (kind, column group, row): 0 Z·ΔW, 1 |Z|² or Σ Z, 2 |X_N|²
  static constexpr uint32_t PART = Dm::WB;
  // ΔW_n of each worker thread in binary16, chunk-slot-major (16 B per thread and slot)
  static constexpr int NSLOT = ((Dm::Dp / 8 > Dm::Wp / 8 ? Dm::Dp / 8 : Dm::Wp / 8) + kFwdGroups - 1) /
                               kFwdGroups;
  static constexpr uint32_t DWS = PART + 3 * kFwdGroups * 128 * 4;
  static constexpr uint32_t BARS = DWS + NSLOT * kFwdWorkers * 16;
  // mbarriers: 0 chain GEMM commits, 1-3 weight images W̃1, W̃2, W̃3
  static constexpr int NBARS = 4;
  static constexpr uint32_t TSLOT = BARS + NBARS * 8;
  static constexpr uint32_t BYTES = TSLOT + 16;
  // the Philox round 0-2 table (fwd_philox_table): NQ x N uint4 rows, then NQ x N words
  static constexpr int NQ = Dm::Dp / 4;
  static constexpr uint32_t TAB = (BYTES + 15u) & ~15u;
  static constexpr uint32_t tab_bytes(int n_steps) { return (uint32_t)NQ * (uint32_t)n_steps * 20u; }
  // tensor memory: the fp32 accumulator, the bf16 A operand of G2/G3 (H1, H2)
  // and that of G1 (X̃_n; no shared-memory operand, so no proxy fence on the
  // workers' path)
  static constexpr uint32_t T_H = 128, T_X = 192, TCOLS = 256;
  static_assert(T_H + Dm::Wp / 2 <= T_X && T_X + Dm::Dp / 2 <= TCOLS, "TMEM budget");
};

// ---------------------------------------------------------------- control warp
template <int D, int W>
__device__ __forceinline__ void fwd_control(const PassArgs& a, int64_t total, uint8_t* sm,
                                            uint32_t tm, int lane) {
  using Dm = Dims<D, W>;
  using L = FwdSmem<D, W>;
  constexpr int Dp = Dm::Dp, Wp = Dm::Wp;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::BARS);
  uint64_t* bg = bars;
  uint64_t* wb = bars + 1;
  const int N = a.N;
  const bool lead = lane == 0;
  const uint8_t* wsrc = static_cast<const uint8_t*>(a.wpack);
  auto reload = [&](int k, int64_t s) {   // weight matrix k (W̃1, W̃2, W̃3) of step s mod N
    if (!lead) return;
    const uint32_t bytes = k == 0 ? Dm::W1B : k == 1 ? Dm::W2B : Dm::W3B;
    const uint32_t off = k == 0 ? L::W1 : k == 1 ? L::W2 : L::W3;
    const uint8_t* src = wsrc + (size_t)((uint32_t)s % (uint32_t)N) * Dm::WB + off;
    mbar_expect_tx(&wb[k], bytes);
    for (uint32_t o = 0; o < bytes; o += 16384u)
      bulk_g2s(sm + off + o, src + o, min(16384u, bytes - o), &wb[k]);
  };
  if (total <= 0) return;
  for (int k = 0; k < 3; ++k) reload(k, 0);
  constexpr uint32_t I1 = idesc_bf16(128, Wp, false, false);
  constexpr uint32_t I3 = idesc_bf16(128, Dp, false, false);
  unsigned long long* const clk = (a.clk && blockIdx.x == 0 && lead) ? a.clk : nullptr;
  for (int64_t s = 0; s < total; ++s) {
    const uint32_t wp = (uint32_t)(s & 1);   // phase of the weight barriers for step s
    named_sync(kBarX, kFwdThreads);          // X̃_n written; E3 of the previous step done
    if (s < 64) BSDE_STAMP(clk, s * 16 + 12);
    if (lead) {
      mbar_wait(&wb[0], wp);
      tc_after();
      gemm_ta(tm, tm + L::T_X, kmaj(sm + L::W1, Dp), Dp / 16, I1, false);
      mma_commit(bg);
    }
    if (s > 0) reload(2, s);                 // G3 of step s-1 has completed: W̃3 -> step s
    __syncwarp();
    named_sync(kBarE1, kFwdThreads);         // H1 in TMEM (so G1 has completed)
    if (s < 64) BSDE_STAMP(clk, s * 16 + 13);
    if (lead) {
      mbar_wait(&wb[1], wp);
      tc_after();
      gemm_ta(tm, tm + L::T_H, kmaj(sm + L::W2, Wp), Wp / 16, I1, false);
      mma_commit(bg);
    }
    if (s + 1 < total) reload(0, s + 1);     // G1 of step s has completed: W̃1 -> step s+1
    __syncwarp();
    named_sync(kBarE2, kFwdThreads);         // H2 in TMEM (G2 has completed)
    if (s < 64) BSDE_STAMP(clk, s * 16 + 14);
    if (lead) {
      mbar_wait(&wb[2], wp);
      tc_after();
      gemm_ta(tm, tm + L::T_H, kmaj(sm + L::W3, Wp), Wp / 16, I3, false);
      mma_commit(bg);
    }
    if (s + 1 < total) reload(1, s + 1);     // G2 of step s has completed: W̃2 -> step s+1
    __syncwarp();
  }
}

// CPL: coupled multilevel paths (a.cpl > 1); MULT: Black-Scholes multiplicative
// noise.  Both are compile-time so that the hot instance carries neither.
template <int D, int W, bool CPL, bool MULT, bool TAB>
__global__ void __launch_bounds__(kFwdThreads, 1) k_fwd_tc(PassArgs a, int ntiles) {
  constexpr bool use_tab = TAB && !CPL;
  using Dm = Dims<D, W>;
  using L = FwdSmem<D, W>;
  constexpr int Dp = Dm::Dp, Wp = Dm::Wp, NCD = Dp / 8, NCW = Wp / 8;
  constexpr int G = kFwdGroups;
  constexpr int NS = ((NCD > NCW ? NCD : NCW) + G - 1) / G;   // chunk slots per worker
  constexpr int NB = 2 * NS;                                   // Philox blocks per worker
#if defined(BSDE_FWD_S1) && defined(BSDE_FWD_S2)   // experiment builds: other splits at d = 100
  constexpr int S1 = NB >= 9 ? BSDE_FWD_S1 : NB / 3, S2 = NB >= 9 ? BSDE_FWD_S2 : 2 * NB / 3;
#else
  // slices [0,S1) [S1,S2) [S2,NB): 4 / 3 / 3 blocks at d = 100 (NB = 10; the front-loaded
  // split covers G1, whose wait was the longest, and measured 1.6% faster than 3 / 3 / 4,
  // profiles/r02_experiments.md), thirds for the small test shapes
  constexpr int S1 = NB >= 9 ? (2 * NB + 2) / 5 : NB / 3, S2 = NB >= 9 ? (7 * NB + 5) / 10 : 2 * NB / 3;
#endif
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::BARS);
  uint64_t* bg = bars;          // chain GEMM commits (3 per step, in order)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::TSLOT);
  float* part = reinterpret_cast<float*>(sm + L::PART);
  __shared__ double lred[kFwdWorkerWarps];
  __shared__ float gred[kFwdWorkerWarps];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    for (int i = 0; i < L::NBARS; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tslot, L::TCOLS);
  uint4* const tab4 = use_tab ? reinterpret_cast<uint4*>(sm + L::TAB) : nullptr;
  uint32_t* const tabE = use_tab ? reinterpret_cast<uint32_t*>(sm + L::TAB + (uint32_t)L::NQ * a.N * 16u) : nullptr;
  if (use_tab) fwd_philox_table(tab4, tabE, L::NQ, a.N, a.eval ? a.eval_it : a.state->it, a.k0, a.k1);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tm = *tslot;
  const int N = a.N;
  const bool store = !a.eval;
  const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  double lsum = 0.0;
  float dy0 = 0.0f;

  if (warp == kFwdWorkerWarps) {
    fwd_control<D, W>(a, (int64_t)my_tiles * N, sm, tm, lane);
  } else {
    // warp group gw = warp / 4 and column group g = (gw + 1) mod 3.  At d = 100 the 25
    // Philox blocks of a path-step split 9 / 8 / 8 over the column groups: the 9-block
    // share goes to the highest warp ids (gw = 2, which the schedulers issue first), the
    // Y recursion to gw = 1, and the lowest-priority group carries neither
#ifndef BSDE_FWD_GROT   // experiment builds: other group rotations / Y-work placements
#define BSDE_FWD_GROT 1
#endif
#ifndef BSDE_FWD_YGW
#define BSDE_FWD_YGW 1
#endif
    const int q = warp & 3, gw = warp >> 2, g = (gw + BSDE_FWD_GROT) % kFwdGroups;
    const bool ywork = gw == BSDE_FWD_YGW;
    const int row = 32 * q + lane;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const uint32_t acc = tm + lane_off, hT = tm + L::T_H + lane_off, xT = tm + L::T_X + lane_off;
    const uint32_t it = a.eval ? a.eval_it : a.state->it;
    uint8_t* xst = static_cast<uint8_t*>(a.xpack);
    uint8_t* dst = static_cast<uint8_t*>(a.dwpack);
    const uint32_t roff = (row >> 3) * (Dp * 16) + (row & 7) * 16;   // row's offset in an image
    constexpr bool mult = MULT;
    const bool hjb = a.problem == kHJB;
    uint4* const dws = reinterpret_cast<uint4*>(sm + L::DWS) + t;   // this thread's ΔW_n slots
    // slot i of this worker is column chunk c = g + 3i (warp-uniform predicates)
    auto chunk = [&](int i) { return g + G * i; };
    unsigned long long* const clk = (a.clk && blockIdx.x == 0 && t == 0) ? a.clk : nullptr;
    uint32_t gph = 0;   // parity of the next chain-GEMM completion
    int64_t s = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t mloc = (int64_t)tile * 128 + row;
      const bool valid = mloc < a.B_local;
      const uint32_t mg = (uint32_t)(a.m0 + mloc);
      float X[8 * NS];
#pragma unroll
      for (int i = 0; i < 8 * NS; ++i) X[i] = a.x0;
      float Y = a.params[0];   // Y and P are carried by the Y-work warp group (ywork)
      float P = 1.0f;          // prefix product P_{n+1} of the ā factors (per_step_abar problems)
      // X̃_n chunk i from X (bf16, constant 1 in column D)
      auto xchunk = [&](int i) {
        const int c = chunk(i);
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          v[e] = col_lt3(g, i, e, D) ? X[8 * i + e] : (8 * c + e == D ? 1.0f : 0.0f);
        return make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
      };
      // X̃_n -> the TMEM operand of G1 (bf16 pairs, 4 columns per chunk)
      auto put_x = [&]() {
#pragma unroll
        for (int i = 0; i < NS; ++i)
          if (chunk_lt3(g, i, NCD)) tmem_st4(xT + 4u * chunk(i), xchunk(i));
        tmem_wait_st();
        tc_before();
      };
      // chunks [I0, I1) of X̃ -> the G1 operand without waiting for the stores: a chunk
      // of X_{n+1} is final once its two Philox blocks are in (chunk i: blocks 2i, 2i+1),
      // and the operand columns are free once G1 of step n has completed (before E1), so
      // the stores are spread over the step and one tcgen05.wait::st in E3 covers them
      auto put_chunks = [&](auto i0c, auto i1c) {
        constexpr int I0 = decltype(i0c)::value, I1 = decltype(i1c)::value;
#pragma unroll
        for (int i = I0; i < I1; ++i)
          if (chunk_lt3(g, i, NCD)) tmem_st4(xT + 4u * chunk(i), xchunk(i));
      };
      constexpr int C1 = S1 / 2, C2 = S2 / 2;   // chunks final after slice 1 / slice 2
      // Y_{n+1} (and P_{n+1}) from the E3 partial sums of step n
      auto finish_y = [&](int n) {
        float cz = 0.f, z2 = 0.f;
#pragma unroll
        for (int k = 0; k < G; ++k) {
          cz += part[(0 * G + k) * 128 + row];
          z2 += part[(1 * G + k) * 128 + row];
        }
        if (store && per_step_abar(a.problem)) {
          P *= 1.0f - a.dt * driver_dfdy(a.problem, Y);
          if (valid) a.Pstore[(int64_t)n * a.B_local + mloc] = P;
        }
        Y = Y - driver_f(a.problem, Y, z2, z2, a.lam) * a.dt + cz;
      };
      put_x();
      named_arrive(kBarX, kFwdThreads);
      // this row's 16-byte chunks in the global images of step n (advanced per step)
      uint8_t* ximg = xst + (size_t)tile * Dm::XB + roff;
      uint8_t* dimg = dst + (size_t)tile * Dm::XB + roff;
      const size_t istep = (size_t)ntiles * Dm::XB;
      for (int n = 0; n < N; ++n, ++s, ximg += istep, dimg += istep) {
        if (s < 64) BSDE_STAMP(clk, s * 16 + 0);
        uint32_t dwh[2 * NB];   // ΔW_n of this worker's columns, binary16 pairs (R17), until
                                // the chunk is complete and parked in shared memory
        // blocks [b0, b1) of ΔW_n: a2 X_{n+1} = X_n + √2 ΔW_n (Black-Scholes:
        // X_n + σ X_n ⊙ ΔW_n) at once, ΔW_n kept as fp16 pairs.  The global
        // images for the adjoint are spread over the slices: X̃_n of a chunk
        // before the slice that starts to advance it, ΔW_n of a chunk once complete.
        auto slice = [&](auto b0c, auto b1c) {
          constexpr int b0 = decltype(b0c)::value, nb = decltype(b1c)::value - b0;
          if constexpr (nb > 0) {
            if (store) {
#pragma unroll
              for (int i = (b0 + 1) / 2; 2 * i < b0 + nb; ++i)
                if (chunk_lt3(g, i, NCD))
                  *reinterpret_cast<uint4*>(ximg + chunk(i) * 128) = xchunk(i);
            }
            // a2 and ΔW_n bookkeeping of block b from its four increments
            auto put_block = [&](int b, const float* z) {
              const int i = b / 2, h = b % 2;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (col_lt3(g, i, 4 * h + e, D)) {
                  float& x = X[8 * i + 4 * h + e];
                  x = mult ? fmaf(kBSSigma * z[e], x, x) : fmaf(kSqrt2, z[e], x);
                }
              dwh[2 * b] = pack_h2(z[0], z[1]);
              dwh[2 * b + 1] = pack_h2(z[2], z[3]);
              if (h == 1 && chunk_lt3(g, i, NCD)) {   // chunk complete: smem copy for E3, image
                const uint4 u = make_uint4(dwh[4 * i], dwh[4 * i + 1], dwh[4 * i + 2], dwh[4 * i + 3]);
                dws[i * kFwdWorkers] = u;
                if (store) *reinterpret_cast<uint4*>(dimg + chunk(i) * 128) = u;
              }
            };
            auto gen = [&](auto bc, auto& z) {   // z: float[4k], blocks bb .. bb+k-1
              constexpr int bb = decltype(bc)::value, k = sizeof(z) / sizeof(float) / 4;
              gen_blocks<D, bb, k, CPL, use_tab>(g, mg, (uint32_t)n, it, a.k0, a.k1, a.sqrt_dt_f, z, a.cpl, tab4, tabE);
            };
            // blocks valid for every column group: one interleaved group
            constexpr int bv = blk_prefix(b0, b0 + nb, D);
            if constexpr (bv > b0) {
              float z[4 * (bv - b0)];
              gen(Int<b0>{}, z);
#pragma unroll
              for (int j = 0; j < bv - b0; ++j) put_block(b0 + j, z + 4 * j);
            }
            // the rest one at a time behind a warp-uniform branch (0 where past D)
            auto tail = [&](auto bc) {
              constexpr int bb = decltype(bc)::value;
              if constexpr (bb < b0 + nb) {
                float z[4] = {0.f, 0.f, 0.f, 0.f};
                if constexpr (!blk_none(bb, D)) {
                  if (col_lt3(g, bb / 2, 4 * (bb % 2), D)) gen(Int<bb>{}, z);
                }
                put_block(bb, z);
              }
            };
            tail(Int<bv>{});
            tail(Int<bv + 1>{});
            tail(Int<bv + 2>{});
            tail(Int<bv + 3>{});
            static_assert(bv + 4 >= b0 + nb, "slice tail longer than four blocks");
          }
        };
        // ---- slice 1 (behind G1); E1: H1 = ReLU(A1) -> TMEM operand
        slice(Int<0>{}, Int<S1>{});
        if (s < 64) BSDE_STAMP(clk, s * 16 + 1);
        mbar_wait(bg, gph);
        gph ^= 1;
        tc_after();
        if (s < 64) BSDE_STAMP(clk, s * 16 + 2);
#pragma unroll
        for (int i0 = 0; i0 < NS; i0 += NS) {   // all chunks' loads in flight, one wait
          uint32_t r[NS][8];
#pragma unroll
          for (int k = 0; k < NS; ++k)
            if (i0 + k < NS && chunk_lt3(g, i0 + k, NCW)) tmem_ld8_nowait(acc + 8u * chunk(i0 + k), r[k]);
          tmem_ld_wait();
          if (s < 64) BSDE_STAMP(clk, s * 16 + 15);
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            if (i0 + k >= NS || !chunk_lt3(g, i0 + k, NCW)) continue;
            reg_fence8(r[k]);
            const float* v = reinterpret_cast<const float*>(r[k]);
            tmem_st4(hT + 4u * chunk(i0 + k),
                     make_uint4(relu_pack2(v[0], v[1]), relu_pack2(v[2], v[3]),
                                relu_pack2(v[4], v[5]), relu_pack2(v[6], v[7])));
          }
        }
#ifdef BSDE_E1DETAIL
        if (s < 64) BSDE_STAMP(clk, s * 16 + 10);
#endif
        tmem_wait_st();
        tc_before();
        named_arrive(kBarE1, kFwdThreads);
#ifdef BSDE_E1DETAIL
        if (s < 64) BSDE_STAMP(clk, s * 16 + 11);
#endif
        if (ywork && n > 0) finish_y(n - 1);   // E3 partials of step n-1 are complete
        if (n + 1 < N) put_chunks(Int<0>{}, Int<C1>{});
        if (s < 64) BSDE_STAMP(clk, s * 16 + 3);
        // ---- slice 2 (behind G2); E2: H2 = H1 + ReLU(A2) in bf16x2 arithmetic (R17)
        slice(Int<S1>{}, Int<S2>{});
        if (n + 1 < N) put_chunks(Int<C1>{}, Int<C2>{});
        if (s < 64) BSDE_STAMP(clk, s * 16 + 4);
        mbar_wait(bg, gph);
        gph ^= 1;
        tc_after();
        if (s < 64) BSDE_STAMP(clk, s * 16 + 5);
#pragma unroll
        for (int i0 = 0; i0 < NS; i0 += 3) {   // E2 holds two registers sets: rounds of 3
          uint32_t r[3][8], h[3][4];
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (i0 + k < NS && chunk_lt3(g, i0 + k, NCW)) {
              tmem_ld8_nowait(acc + 8u * chunk(i0 + k), r[k]);
              tmem_ld4_nowait(hT + 4u * chunk(i0 + k), h[k]);
            }
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            if (i0 + k >= NS || !chunk_lt3(g, i0 + k, NCW)) continue;
            reg_fence8(r[k]);
            reg_fence4(h[k]);
            const float* v = reinterpret_cast<const float*>(r[k]);
            tmem_st4(hT + 4u * chunk(i0 + k),
                     make_uint4(bf2_add(h[k][0], relu_pack2(v[0], v[1])),
                                bf2_add(h[k][1], relu_pack2(v[2], v[3])),
                                bf2_add(h[k][2], relu_pack2(v[4], v[5])),
                                bf2_add(h[k][3], relu_pack2(v[6], v[7]))));
          }
        }
        tmem_wait_st();
        tc_before();
        named_arrive(kBarE2, kFwdThreads);
        if (s < 64) BSDE_STAMP(clk, s * 16 + 6);
        // ---- slice 3 (behind G3)
        slice(Int<S2>{}, Int<NB>{});
        if (n + 1 < N) put_chunks(Int<C2>{}, Int<NS>{});   // the rest of X̃_{n+1}, behind G3
        if (s < 64) BSDE_STAMP(clk, s * 16 + 7);
        // ---- E3: partial sums of Z·ΔW (|Z|² for HJB, Σ Z for Black-Scholes) over
        // this worker's columns, with the binary16 ΔW_n (R17)
        mbar_wait(bg, gph);
        gph ^= 1;
        tc_after();
        if (s < 64) BSDE_STAMP(clk, s * 16 + 8);
        {
          float cz[2] = {0.f, 0.f}, z2[2] = {0.f, 0.f};
          constexpr int RZ = NS;   // every chunk's load in flight, one wait
#pragma unroll
          for (int i0 = 0; i0 < NS; i0 += RZ) {
            uint32_t r[RZ][8];
#pragma unroll
            for (int k = 0; k < RZ; ++k)
              if (i0 + k < NS && col_lt3(g, i0 + k, 0, D)) tmem_ld8_nowait(acc + 8u * chunk(i0 + k), r[k]);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < RZ; ++k) {
              const int i = i0 + k;
              if (i >= NS || !col_lt3(g, i, 0, D)) continue;
              reg_fence8(r[k]);
              const float* zv = reinterpret_cast<const float*>(r[k]);
              float dwv[8];
              unpack_dw(dws[i * kFwdWorkers], dwv);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (col_lt3(g, i, e, D)) {
                  cz[e & 1] = fmaf(zv[e], dwv[e], cz[e & 1]);
                  if (hjb) z2[e & 1] = fmaf(zv[e], zv[e], z2[e & 1]);
                  else if (mult) z2[e & 1] += zv[e];
                }
            }
          }
#ifndef BSDE_E1DETAIL
          if (s < 64) BSDE_STAMP(clk, s * 16 + 10);
#endif
          part[(0 * G + g) * 128 + row] = cz[0] + cz[1];
          part[(1 * G + g) * 128 + row] = z2[0] + z2[1];
        }
        tc_before();
#ifndef BSDE_E1DETAIL
        if (s < 64) BSDE_STAMP(clk, s * 16 + 11);
#endif
        if (n + 1 < N) {   // X̃_{n+1} complete: G1 of step n+1 may start
          tmem_wait_st();
          tc_before();
          named_arrive(kBarX, kFwdThreads);
        }
        if (s < 64) BSDE_STAMP(clk, s * 16 + 9);
      }
      // ---- a5 (tile tail): Y_N, R = Y_N - g(X_N), loss, ā_N (times P_N), dY0 = ā_0
      {
        float sx = 0.0f;   // |X_N|² partial of this worker's columns
#pragma unroll
        for (int i = 0; i < NS; ++i)
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (col_lt3(g, i, e, D)) sx = fmaf(X[8 * i + e], X[8 * i + e], sx);
        part[(2 * G + g) * 128 + row] = sx;
      }
      named_sync(kBarTail, kFwdWorkers);
      if (ywork) {
        finish_y(N - 1);
        if (valid) {
          float xn2 = 0.0f;
#pragma unroll
          for (int k = 0; k < G; ++k) xn2 += part[(2 * G + k) * 128 + row];
          const float R = Y - terminal_g(a.problem, xn2);
          lsum += (double)R * R;
          if (store) {
            a.Rstore[mloc] = R;
            float ab = 2.0f * R * a.inv_B;
            if (per_step_abar(a.problem)) ab *= P;
            a.abar[mloc] = ab;
            dy0 += ab;
          }
        }
      }
      named_sync(kBarTail, kFwdWorkers);   // partials read before they are rewritten
    }
  }
  double lw = lsum;
  float gw = dy0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lw += __shfl_xor_sync(0xffffffffu, lw, o);
    gw += __shfl_xor_sync(0xffffffffu, gw, o);
  }
  if (warp < kFwdWorkerWarps && lane == 0) { lred[warp] = lw; gred[warp] = gw; }
  tc_before();
  __syncthreads();
  if (t == 0) {
    double Ls = 0.0;
    float g0 = 0.0f;
    for (int w = 0; w < kFwdWorkerWarps; ++w) { Ls += lred[w]; g0 += gred[w]; }
    if (a.lpart) {   // deterministic mode: per-CTA partials, summed in order by k_det_reduce
      a.lpart[blockIdx.x] = Ls;
      a.y0part[blockIdx.x] = a.eval ? 0.0f : g0;
    } else {
      if (Ls != 0.0) atomicAdd(a.loss_acc, Ls);
      if (!a.eval && g0 != 0.0f) atomicAdd(a.grad, g0);
    }
  }
  if (warp == 0) {
    tc_after();
    tmem_dealloc(tm, L::TCOLS);
  }
}

}  // namespace tc
}  // namespace bsde
