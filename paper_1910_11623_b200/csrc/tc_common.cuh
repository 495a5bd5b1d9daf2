// tc_common.cuh — sm_100a building blocks of the tcgen05 kernels: PTX wrappers
// (mbarrier, bulk copies, TMEM alloc/ld, tcgen05.mma/commit), shared-memory
// matrix descriptors, and the bf16 operand-image layout.
//
// Operand images: a [R×C] bf16 matrix in the canonical no-swizzle UMMA layout of
// 8x8 core matrices: byte offset(r, c) = (r/8)·(C·16) + (c/8)·128 + (r%8)·16 + (c%8)·2.
//   as a K-major operand (rows = M|N, K = C):  LBO = 128,  SBO = C·16, K-step 256 B
//   as an MN-major operand (M|N = C, K = R):   LBO = C·16, SBO = 128,  K-step C·32 B
// (pinned on the device by tests/test_gpu_tc.py::test_umma_operand_layouts).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>
#ifdef BSDE_WATCHDOG
#include <cstdio>
#endif

namespace bsde {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Blocking phase wait.  try_wait suspends the thread until the phase completes
// or the time hint (1 ms) elapses, so waiting warps do not spin on the issue
// slots the working warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
#ifdef BSDE_WATCHDOG
// debug builds: a phase wait that reports (barrier offset, parity, block, thread) and
// traps after ~2 s instead of hanging
static __device__ __noinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, int tag) {
  for (long long i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(1000u) : "memory");
    if (ok) return;
    if (i == 2000000 && (threadIdx.x & 31) == 0) {
      printf("WATCHDOG tag %d bar %p parity %u block %d thread %d\n", tag, bar, parity, blockIdx.x, threadIdx.x);
      asm volatile("trap;");
    }
  }
}
#define mbar_wait(b, p) mbar_wait_wd((b), (p), __LINE__)
#endif
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// barrier `id` (1..15) over `nthreads` threads (a multiple of 32)
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// signal barrier `id` (counting `nthreads`) without waiting for it
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// non-blocking probe of a phase
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// prefetch [src, src+bytes) into L2 (no shared-memory destination)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// 16-byte asynchronous global -> shared copy by the calling thread (LDGSTS):
// never blocks the thread; completion via cp_async_wait_all().
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D (+)= A·B with A read from tensor memory (kind::f16: row r of A in lane r,
// bf16 pairs (k, k+1) packed per 32-bit column, low half = even k; one K=16
// step spans 8 columns).
__device__ __forceinline__ void mma_bf16_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// four 32-bit columns [taddr, taddr+4) of the calling thread's lane
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint4& u) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 16 consecutive fp32 columns of the calling thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Four 8-column chunks of the calling thread's lane, at column offsets
// c0, c0+32, c0+64, c0+96 (the chunks g, g+4, g+8, g+12 of column group g),
// issued back to back with a single wait.
__device__ __forceinline__ void tmem_ld4x8(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%33];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%34];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [%35];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr), "r"(taddr + 32u), "r"(taddr + 64u), "r"(taddr + 96u)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Two 8-column chunks of the calling thread's lane at column offsets c0, c0+32.
__device__ __forceinline__ void tmem_ld2x8(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%16];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%17];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr), "r"(taddr + 32u)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 8 consecutive fp32 columns of the calling thread's lane, without the wait:
// issue several, then tmem_ld_wait() and reg_fence8() on each destination.
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// orders later uses of r after the preceding tmem_ld_wait()
__device__ __forceinline__ void reg_fence8(uint32_t (&r)[8]) {
  asm volatile("" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
               "+r"(r[6]), "+r"(r[7]));
}
__device__ __forceinline__ void tmem_ld4_nowait(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void reg_fence4(uint32_t (&r)[4]) {
  asm volatile("" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]));
}
// chunks c = c0 + 2i (i < NC) of 8 columns each from TMEM lane address base
template <int NC>
__device__ __forceinline__ void tmem_ld_chunks2(uint32_t base, int c0, float (&v)[NC][8]) {
  uint32_t r[NC][8];
#pragma unroll
  for (int i = 0; i < NC; ++i) tmem_ld8_nowait(base + 8u * (uint32_t)(c0 + 2 * i), r[i]);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    reg_fence8(r[i]);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[i][e] = __uint_as_float(r[i][e]);
  }
}

// chunks c0 + i (i < NC, only those with i < nvalid) of 8 columns each from TMEM
template <int NC>
__device__ __forceinline__ void tmem_ld_chunks(uint32_t base, float (&v)[NC][8], int nvalid) {
  uint32_t r[NC][8];
#pragma unroll
  for (int i = 0; i < NC; ++i)
    if (i < nvalid) tmem_ld8_nowait(base + 8u * (uint32_t)i, r[i]);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    if (i < nvalid) {
      reg_fence8(r[i]);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[i][e] = __uint_as_float(r[i][e]);
    }
  }
}

// The calling thread's chunks g + 4i (i < 4) that exist in an NC-chunk matrix
// (columns 8(g + 4i) .. +7 from taddr = first chunk of the thread); chunks past
// the matrix are not read (they may lie past the allocation) and read as 0.
__device__ __forceinline__ void tmem_ld_g4(uint32_t taddr, int g, int NC, float (&v)[32]) {
  uint32_t r[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (g + 4 * i < NC) tmem_ld8_nowait(taddr + 32u * i, r[i]);
    else
#pragma unroll
      for (int e = 0; e < 8; ++e) r[i][e] = 0u;
  }
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    reg_fence8(r[i]);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[8 * i + e] = __uint_as_float(r[i][e]);
  }
}

// clock64() phase tracing of CTA 0 (tools/phase_clocks.py): compiled in only
// with -DBSDE_PHASE_CLOCKS, so the product kernels carry no clock reads.
#ifdef BSDE_PHASE_CLOCKS
#define BSDE_STAMP(ptr, idx) do { if (ptr) (ptr)[idx] = clock64(); } while (0)
#else
#define BSDE_STAMP(ptr, idx) do { (void)(ptr); } while (0)
#endif

// mbarrier phase wait that suspends the thread for at most `ns` nanoseconds;
// returns whether the phase completed
__device__ __forceinline__ bool mbar_try_wait_ns(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

template <int I>
struct Int {
  static constexpr int value = I;
};

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);   // version 1, no swizzle
}
// kind::f16 instruction descriptor: D fp32 (bit 4), A/B bf16 (bits 7, 10), A/B
// major (bits 15, 16), N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct Opnd {
  uint32_t base, lbo, sbo, kstep;
};
__device__ __forceinline__ Opnd kmaj(const void* img, int C) {
  return Opnd{smem_u32(img), 128u, (uint32_t)C * 16u, 256u};
}
__device__ __forceinline__ Opnd mnmaj(const void* img, int C) {
  return Opnd{smem_u32(img), (uint32_t)C * 16u, 128u, (uint32_t)C * 32u};
}
// D (+)= A·B over ksteps·16 of K; issued by one thread.
// The descriptors are built once; a K step only advances the 14-bit start
// address field (bits 0-13, in 16-byte units), which cannot carry out for
// operands inside the 227 KB of shared memory.
__device__ __forceinline__ void gemm(uint32_t d_tmem, Opnd A, Opnd B, int ksteps, uint32_t idesc,
                                     bool accumulate) {
  const uint64_t a0 = sdesc(A.base, A.lbo, A.sbo), b0 = sdesc(B.base, B.lbo, B.sbo);
  const uint32_t ai = A.kstep >> 4, bi = B.kstep >> 4;
#pragma unroll
  for (int k = 0; k < ksteps; ++k)
    mma_bf16(d_tmem, a0 + (uint64_t)(k * ai), b0 + (uint64_t)(k * bi), idesc,
             (k > 0 || accumulate) ? 1u : 0u);
}

// D (+)= A·B over ksteps·16 of K with A in tensor memory at column a_tmem.
__device__ __forceinline__ void gemm_ta(uint32_t d_tmem, uint32_t a_tmem, Opnd B, int ksteps,
                                        uint32_t idesc, bool accumulate) {
  const uint64_t b0 = sdesc(B.base, B.lbo, B.sbo);
  const uint32_t bi = B.kstep >> 4;
#pragma unroll
  for (int k = 0; k < ksteps; ++k)
    mma_bf16_ta(d_tmem, a_tmem + 8u * k, b0 + (uint64_t)(k * bi), idesc,
                (k > 0 || accumulate) ? 1u : 0u);
}

__host__ __device__ constexpr int pad16(int x) { return (x + 15) / 16 * 16; }

template <int D, int W>
struct Dims {
  static constexpr int Dp = pad16(D + 1);    // + constant-1 column (folded bias)
  static constexpr int Wp = pad16(W + 1);
  static constexpr int KM = Dp > Wp ? Dp : Wp;
  static constexpr uint32_t W1B = Wp * Dp * 2, W2B = Wp * Wp * 2, W3B = Dp * Wp * 2;
  static constexpr uint32_t WB = W1B + W2B + W3B;          // one step's weight images
  static constexpr uint32_t XB = 128u * Dp * 2;            // X operand image of one tile
  // an M=128 MN-major operand over a C-column image reads (128 - C)/8 core-matrix
  // columns past each row group (feeding D rows that are never read): pad for it
  static constexpr int CMIN = Dp < Wp ? Dp : Wp;
  static constexpr uint32_t ACT = 128u * KM * 2 + (128 - CMIN) / 8 * 128 + 256;
  static_assert(Dp <= 128 && Wp <= 128, "tcgen05 tiles need d+1 <= 128 and w+1 <= 128");
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// bf16x2 {lo = ReLU(a), hi = ReLU(b)} (RNE), one instruction
__device__ __forceinline__ uint32_t relu_pack2(float a, float b) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(b), "f"(a));
  return d;
}
// bf16x2 sum (RNE)
__device__ __forceinline__ uint32_t bf2_add(uint32_t x, uint32_t y) {
  uint32_t d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
  return d;
}
// per-half 0xFFFF where the bf16 half is non-zero, for halves >= +0 (ReLU
// outputs): h + 0x7FFF sets bit 15 of the half iff h != 0 without carrying
// out of it, and PRMT replicates that bit over the half.
__device__ __forceinline__ uint32_t nz_mask2(uint32_t w) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(d) : "r"(w + 0x7FFF7FFFu));
  return d;
}
__device__ __forceinline__ void st_chunk_u4(uint8_t* img, int row, int chunk, int C, const uint4& u) {
  *reinterpret_cast<uint4*>(img + (row >> 3) * (C * 16) + chunk * 128 + (row & 7) * 16) = u;
}

// row `row`, columns [8·chunk, 8·chunk + 8) of an image with C columns
__device__ __forceinline__ void st_chunk(uint8_t* img, int row, int chunk, int C, const float* v) {
  uint4 u;
  u.x = pack2(v[0], v[1]);
  u.y = pack2(v[2], v[3]);
  u.z = pack2(v[4], v[5]);
  u.w = pack2(v[6], v[7]);
  *reinterpret_cast<uint4*>(img + (row >> 3) * (C * 16) + chunk * 128 + (row & 7) * 16) = u;
}
__device__ __forceinline__ void ld_chunk(const uint8_t* img, int row, int chunk, int C, float* v) {
  const uint4 u =
      *reinterpret_cast<const uint4*>(img + (row >> 3) * (C * 16) + chunk * 128 + (row & 7) * 16);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

}  // namespace tc
}  // namespace bsde
