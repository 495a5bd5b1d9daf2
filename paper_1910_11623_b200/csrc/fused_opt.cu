// fused_opt.cu — SURVEY §8(f) NEXT-4: the gradient reduce-scatter, Adam on this
// rank's 1/world shard and the all-gather of the updated parameters as ONE kernel over
// peer memory (NVLink loads and stores through CUDA IPC mappings), chained after the
// adjoint in the captured step graph.  It replaces the NCCL allreduce (or
// reduce-scatter / all-gather) + k_check + k_adam of enqueue_step
// (BASELINE north_star (e); "shard gradients are summed before adam_step
// ... deterministic fixed-order reduction mode").
//
// Rank r owns the parameter indices [r·S, (r+1)·S) (S = shard, a multiple of 4).
//   x-rank barrier 1   every rank's gradient (and Σ R²) is complete
//   reduce             g_i = Σ_q grad_q[i] in rank order (deterministic), i in the
//                      shard, written in place (no peer reads this rank's shard of
//                      its own buffer); loss = Σ_q lossum_q / B; finite checks
//   x-rank barrier 2   the divergence flags are exchanged (any rank diverged: skip)
//   Adam + gather      θ_i, m_i, v_i updated (R6), θ_i stored into every rank's
//                      parameter buffer (peer stores)
//   x-rank barrier 3   all parameters are in place before the weight images are packed
// Cross-rank barriers are monotone counters in each rank's flag buffer incremented by
// every rank with system-scope atomics; grid barriers are a monotone counter in the
// local flag buffer.  The launch index (epoch) lives in DeviceState, so a replayed
// graph needs no new kernel arguments.  Requires all blocks co-resident: one block
// per SM.  At world = 1 the peers are the context itself and the kernel is the
// collective-free Adam step, bit for bit (tests/test_gpu_fused_opt.py).
#include "kernels.cuh"

namespace bsde {
namespace {

constexpr int FT = 512;              // threads per block
constexpr int kGridBars = 4;         // grid barriers per launch
constexpr int kPeerBars = 3;         // cross-rank barriers per launch

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// flags[0]: cross-rank arrivals; flags[1 + q]: rank q's divergence flag;
// flags[16]: grid-barrier counter (local)
__device__ void grid_barrier(unsigned* flags, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&flags[16], 1u);
    while (ld_acquire_sys(&flags[16]) < target) __nanosleep(64);
  }
  __syncthreads();
}

__device__ void peer_barrier(const FusedOptArgs& a, unsigned target) {   // block 0, thread 0
  __threadfence_system();
  for (int q = 0; q < a.world; ++q) atomicAdd_system(a.peer_flags[q], 1u);
  while (ld_acquire_sys(a.peer_flags[a.rank]) < target) __nanosleep(128);
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const void* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(FT, 1) k_fused_opt(FusedOptArgs a) {
  // Every value another block wrote in this launch is read with an acquire load by one
  // thread after a grid barrier and handed to the block through shared memory: plain
  // loads could hit a line the SM's (non-coherent) L1 cached earlier in the launch.
  __shared__ unsigned s_epoch, s_skip;
  __shared__ float s_c1, s_c2;
  unsigned* fl = a.peer_flags[a.rank];
  DeviceState* st = a.state;
  if (threadIdx.x == 0) {
    s_epoch = ld_acquire_gpu(&st->opt_epoch);
    // Adam bias corrections of this step (as k_check): t is written by k_end_step of the
    // previous launch only, so every block derives the same c1, c2 itself
    const int t1 = (int)ld_acquire_gpu(&st->t) + 1;
    s_c1 = (float)(1.0 / (1.0 - pow((double)a.beta1, (double)t1)));
    s_c2 = (float)(1.0 / (1.0 - pow((double)a.beta2, (double)t1)));
  }
  __syncthreads();
  const unsigned e = s_epoch, G = (unsigned)gridDim.x, W = (unsigned)a.world;
  unsigned gb = 0;   // grid barriers passed in this launch
  auto gbar = [&]() { grid_barrier(fl, (e * kGridBars + (++gb)) * G); };
  // 1: every rank's gradient and loss sum are complete
  if (blockIdx.x == 0 && threadIdx.x == 0) peer_barrier(a, (e * kPeerBars + 1) * W);
  gbar();
  // reduce this rank's shard in rank order, in place; finite check
  const int64_t lo = (int64_t)a.rank * a.shard, hi = lo + a.shard < a.np ? lo + a.shard : a.np;
  bool bad = false;
  for (int64_t i = lo + blockIdx.x * (int64_t)FT + threadIdx.x; i < hi; i += (int64_t)G * FT) {
    float g = 0.0f;
    for (int q = 0; q < a.world; ++q) g += __ldcg(a.peer_grad[q] + i);
    a.peer_grad[a.rank][i] = g;
    bad |= !isfinite(g);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->diverged, 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // the global loss (fixed order)
    double ls = 0.0;
    for (int q = 0; q < a.world; ++q) ls += __ldcg(&a.peer_state[q]->loss_sum);
    st->loss_sum = ls;
    const double loss = ls * a.inv_B;
    st->loss_last = loss;
    if (!(loss <= 1e12)) atomicOr(&st->diverged, 1);
    st->c1 = s_c1;
    st->c2 = s_c2;
  }
  gbar();
  // 2: the divergence decision is the OR over the ranks
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned mine = ld_acquire_gpu(&st->diverged);
    for (int q = 0; q < a.world; ++q) atomicExch_system(&a.peer_flags[q][1 + a.rank], mine);
    peer_barrier(a, (e * kPeerBars + 2) * W);
    unsigned any = 0;
    for (int q = 0; q < a.world; ++q) any |= ld_acquire_sys(&fl[1 + q]);
    st->diverged = any ? 1 : 0;
  }
  gbar();
  if (threadIdx.x == 0) s_skip = ld_acquire_gpu(&st->diverged);
  __syncthreads();
  // Adam on the shard (R6; skipped on divergence) and the all-gather by peer stores
  if (!s_skip) {
    const float c1 = s_c1, c2 = s_c2, b1 = a.beta1, b2 = a.beta2, lr = a.lr, eps = a.eps;
    float* p = a.peer_params[a.rank];
    const float* g = a.peer_grad[a.rank];
    for (int64_t i = lo + blockIdx.x * (int64_t)FT + threadIdx.x; i < hi; i += (int64_t)G * FT) {
      const float gg = __ldcg(g + i);
      const float mm = fmaf(b1, a.m[i], (1.0f - b1) * gg);
      const float vv = fmaf(b2, a.v[i], (1.0f - b2) * gg * gg);
      const float pp = p[i] - lr * (mm * c1) / (sqrtf(vv * c2) + eps);
      a.m[i] = mm;
      a.v[i] = vv;
      for (int q = 0; q < a.world; ++q) a.peer_params[q][i] = pp;
    }
  }
  gbar();
  // 3: all shards are in every rank's parameters
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    peer_barrier(a, (e * kPeerBars + 3) * W);
    st->opt_epoch = e + 1;
  }
  gbar();
}

}  // namespace

cudaError_t launch_fused_opt(const FusedOptArgs& a, int sms, cudaStream_t s) {
  k_fused_opt<<<sms, FT, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace bsde
