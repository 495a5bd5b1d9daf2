// aux.cu — initialisation (R7), step bookkeeping, divergence check, fused Adam
// (a8, R6), multilevel prolongation (a9; §3.2 PAPER.md:237-252,
// R14) and the generator test hooks (pin H0).
#include "kernels.cuh"

namespace bsde {
namespace {

constexpr int NT = 256;

__global__ void k_init_params(float* __restrict__ params, int d, int w, int N, uint32_t k0,
                              uint32_t k1, int zero_head, int nais) {
  const NetDims nd{d, w, nais};
  const int64_t P = nd.step_size();
  const int64_t total = 1 + (int64_t)N * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t tid = 0, idx = 0;
    int fan_in = 0, fan_out = 0;
    bool weight = false;
    if (i == 0) {
      tid = 0; idx = 0;
    } else {
      const int64_t n = (i - 1) / P, r = (i - 1) - n * P;
      const uint32_t base = 1u + 3u * (uint32_t)n;
      if (r < nd.off_b1()) { tid = base; idx = (uint32_t)r; fan_in = d; fan_out = w; weight = true; }
      else if (r >= nd.off_W2() && r < nd.off_b2()) {
        tid = base + 1; idx = (uint32_t)(r - nd.off_W2()); fan_in = w; fan_out = w; weight = true;
      } else if (r >= nd.off_W3() && r < nd.off_b3() && !zero_head) {
        tid = base + 2; idx = (uint32_t)(r - nd.off_W3()); fan_in = w; fan_out = d; weight = true;
      } else if (nais && r >= nd.off_B()) {          // B_n of the NAIS block (R25)
        tid = 0x100000u + (uint32_t)n; idx = (uint32_t)(r - nd.off_B()); fan_in = d; fan_out = w;
        weight = true;
      } else {
        params[i] = 0.0f;      // biases (and W3 with a zero head, R7b)
        continue;
      }
    }
    const uint4 x = philox4x32_10(make_uint4(idx >> 2, tid, 0u, kInitStream), k0, k1);
    const uint32_t sel = (idx & 3) == 0 ? x.x : (idx & 3) == 1 ? x.y : (idx & 3) == 2 ? x.z : x.w;
    const float u = unit_from_u32(sel);
    if (!weight) {
      params[i] = u;                                    // Y0 ~ U(0,1)
    } else {
      const float a = sqrtf(6.0f / (float)(fan_in + fan_out));
      params[i] = a * (2.0f * u - 1.0f);                // Xavier-uniform
    }
  }
}

// NAIS-Net projection (R25, SPEC nets.project_R), one CTA per step n:
// f = ‖RᵀR‖_F = (Σ_{i,j} (Σ_r R[r][i] R[r][j])²)^½; if f > 1-ε, R *= ((1-ε)/f)^½.
__global__ void k_nais_project(float* __restrict__ params, int d, int w) {
  const NetDims nd{d, w, 1};
  float* R = params + nd.step_base(blockIdx.x) + nd.off_W2();
  double acc = 0.0;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int i = e / w, j = e - i * w;
    float g = 0.0f;
    for (int r = 0; r < w; ++r) g = fmaf(R[r * w + i], R[r * w + j], g);
    acc += (double)g * g;
  }
  __shared__ double red[NT / 32];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  __shared__ float scale;
  if (threadIdx.x == 0) {
    double f2 = 0.0;
    for (int k = 0; k < NT / 32; ++k) f2 += red[k];
    const double f = sqrt(f2);
    scale = f > 1.0 - kNaisEps ? (float)sqrt((1.0 - kNaisEps) / f) : 1.0f;
  }
  __syncthreads();
  if (scale != 1.0f)
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) R[e] *= scale;
}

// The adjoint accumulates Ā = Σ dA2ᵀ H1 in the W2 slot (the gradient with respect
// to A); A = -RᵀR - εI gives R̄ = -R(Ā + Āᵀ) (R25).  One CTA per step.
__global__ void k_nais_grad(const float* __restrict__ params, float* __restrict__ grad, int d,
                            int w) {
  extern __shared__ float S[];   // [w][w] Ā + Āᵀ
  const NetDims nd{d, w, 1};
  const float* R = params + nd.step_base(blockIdx.x) + nd.off_W2();
  float* G = grad + nd.step_base(blockIdx.x) + nd.off_W2();
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int i = e / w, j = e - i * w;
    S[e] = G[i * w + j] + G[j * w + i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int i = e / w, j = e - i * w;
    float g = 0.0f;
    for (int k = 0; k < w; ++k) g = fmaf(R[i * w + k], S[k * w + j], g);
    G[e] = -g;
  }
}

// Deterministic reduction (cfg.deterministic): one thread per (step, parameter)
// sums the adjoint CTAs' partials in CTA order; block 0 thread 0 also sums the
// forward CTAs' loss and dY0 partials.  CTA c of the adjoint owns items
// [c·items/G, (c+1)·items/G), item = n·ntiles + tile.
__global__ void k_det_reduce(PassArgs a, int fwd_grid, int bwd_grid, int64_t items, int ntiles) {
  const NetDims nd{a.d, a.w, a.nais};
  const int64_t P = nd.step_size();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double L = 0.0;
    float g0 = 0.0f;
    for (int c = 0; c < fwd_grid; ++c) { L += a.lpart[c]; g0 += a.y0part[c]; }
    *a.loss_acc += L;
    if (!a.eval) a.grad[0] += g0;
  }
  if (bwd_grid == 0) return;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < (int64_t)a.N * P;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(id / P);
    const int64_t i = id - (int64_t)n * P;
    // CTAs covering step n: i1(c) > n·ntiles and i0(c) < (n+1)·ntiles
    const int64_t lo_item = (int64_t)n * ntiles, hi_item = lo_item + ntiles;
    int c = max(0, (int)((lo_item * bwd_grid) / items) - 1);
    float v = 0.0f;
    for (; c < bwd_grid; ++c) {
      const int64_t i0 = (int64_t)c * items / bwd_grid, i1 = (int64_t)(c + 1) * items / bwd_grid;
      if (i0 >= hi_item) break;
      if (i1 <= lo_item || i0 >= i1) continue;
      const int seg = n - (int)(i0 / ntiles);
      v += a.dpart[((int64_t)c * a.dseg + seg) * P + i];
    }
    a.grad[nd.step_base(n) + i] = v;
  }
}

__global__ void k_begin_step(DeviceState* st) {
  st->loss_sum = 0.0;
  st->diverged = 0;
}

// Non-finite gradient anywhere, or loss non-finite / > 1e12 ⇒ skip the update.
__global__ void k_check(const float* __restrict__ grad, int64_t n, DeviceState* st,
                        double inv_B, float beta1, float beta2) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(grad[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->diverged, 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double loss = st->loss_sum * inv_B;
    st->loss_last = loss;
    if (!(loss <= 1e12)) atomicOr(&st->diverged, 1);   // also catches NaN
    const int t1 = st->t + 1;
    st->c1 = (float)(1.0 / (1.0 - pow((double)beta1, (double)t1)));
    st->c2 = (float)(1.0 / (1.0 - pow((double)beta2, (double)t1)));
  }
}

// θ ← θ - lr m̂/(√v̂ + ε) with m̂ = m c1, v̂ = v c2 (R6); skipped on divergence.
__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, const DeviceState* st, float lr,
                       float beta1, float beta2, float eps) {
  if (st->diverged) return;
  const float c1 = st->c1, c2 = st->c2;
  const int64_t n4 = n >> 2;
  float4* p4 = reinterpret_cast<float4*>(p);
  float4* m4 = reinterpret_cast<float4*>(m);
  float4* v4 = reinterpret_cast<float4*>(v);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  auto upd = [&](float& pp, float gg, float& mm, float& vv) {
    mm = fmaf(beta1, mm, (1.0f - beta1) * gg);
    vv = fmaf(beta2, vv, (1.0f - beta2) * gg * gg);
    pp -= lr * (mm * c1) / (sqrtf(vv * c2) + eps);
  };
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = p4[i], mm = m4[i], vv = v4[i];
    const float4 gg = __ldg(g4 + i);
    upd(pp.x, gg.x, mm.x, vv.x);
    upd(pp.y, gg.y, mm.y, vv.y);
    upd(pp.z, gg.z, mm.z, vv.z);
    upd(pp.w, gg.w, mm.w, vv.w);
    p4[i] = pp; m4[i] = mm; v4[i] = vv;
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t i = (n4 << 2) + threadIdx.x;
    upd(p[i], g[i], m[i], v[i]);
  }
}

__global__ void k_end_step(DeviceState* st, int advance_it) {
  if (!st->diverged) st->t += 1;
  st->diverged_any |= st->diverged;
  if (advance_it) st->it += 1;
}

// dst (2N steps) from src (N steps); Y0 copied.  mode 0: copy, 1: midpoint.
__global__ void k_prolong(const float* __restrict__ src, float* __restrict__ dst, int64_t P,
                          int N, int mode) {
  const int64_t total = 2LL * N * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / P, r = i - k * P;
    const int64_t c = k >> 1;
    float v = src[1 + c * P + r];
    if (mode == 1 && (k & 1) && c < N - 1) v = 0.5f * (v + src[1 + (c + 1) * P + r]);
    dst[1 + i] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) dst[0] = src[0];
}

__global__ void k_debug_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int64_t count,
                               uint32_t* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint4 x = philox4x32_10(make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]), k0, k1);
  out[4 * i] = x.x; out[4 * i + 1] = x.y; out[4 * i + 2] = x.z; out[4 * i + 3] = x.w;
}

__global__ void k_debug_dw(uint32_t it, int n, int64_t m0, int64_t count, int d, float sqrt_dt,
                           uint32_t k0, uint32_t k1, float* out) {
  const int nq = (d + 3) >> 2;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count * nq) return;
  const int64_t p = i / nq;
  const int q = (int)(i - p * nq);
  const float4 z = normals4((uint32_t)q, (uint32_t)(m0 + p), (uint32_t)n, it, k0, k1);
  const float zz[4] = {z.x, z.y, z.z, z.w};
  for (int k = 0; k < 4; ++k)
    if (4 * q + k < d) out[p * d + 4 * q + k] = sqrt_dt * zz[k];
}

int grid_for(int64_t n) {
  int64_t g = (n + NT - 1) / NT;
  if (g > 148 * 8) g = 148 * 8;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

cudaError_t launch_init_params(float* params, int d, int w, int N, uint32_t k0, uint32_t k1,
                               int zero_head, int nais, cudaStream_t s) {
  const int64_t total = 1 + (int64_t)N * NetDims{d, w, nais}.step_size();
  k_init_params<<<grid_for(total), NT, 0, s>>>(params, d, w, N, k0, k1, zero_head, nais);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && nais) e = launch_nais_project(params, d, w, N, s);   // R25: init projected
  return e;
}

int det_segments(int64_t items, int grid, int ntiles) {
  int best = 1;
  for (int c = 0; c < grid; ++c) {
    const int64_t i0 = (int64_t)c * items / grid, i1 = (int64_t)(c + 1) * items / grid;
    if (i1 > i0) best = max(best, (int)((i1 - 1) / ntiles - i0 / ntiles + 1));
  }
  return best;
}

cudaError_t launch_det_reduce(const PassArgs& a, int fwd_grid, int bwd_grid, int64_t items,
                              int ntiles, cudaStream_t s) {
  const int64_t work = bwd_grid ? (int64_t)a.N * NetDims{a.d, a.w, a.nais}.step_size() : 1;
  k_det_reduce<<<grid_for(work), NT, 0, s>>>(a, fwd_grid, bwd_grid, items, ntiles);
  return cudaGetLastError();
}

cudaError_t launch_nais_project(float* params, int d, int w, int N, cudaStream_t s) {
  k_nais_project<<<N, NT, 0, s>>>(params, d, w);
  return cudaGetLastError();
}

cudaError_t launch_nais_grad(const float* params, float* grad, int d, int w, int N, cudaStream_t s) {
  const size_t smem = (size_t)w * w * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(k_nais_grad, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_nais_grad<<<N, NT, smem, s>>>(params, grad, d, w);
  return cudaGetLastError();
}

cudaError_t launch_begin_step(DeviceState* st, float* grad, int64_t n_grad, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(grad, 0, sizeof(float) * n_grad, s);
  if (e != cudaSuccess) return e;
  k_begin_step<<<1, 1, 0, s>>>(st);
  return cudaGetLastError();
}

cudaError_t launch_check(const float* grad, int64_t n, DeviceState* st, double inv_B,
                         float beta1, float beta2, cudaStream_t s) {
  k_check<<<grid_for(n), NT, 0, s>>>(grad, n, st, inv_B, beta1, beta2);
  return cudaGetLastError();
}

cudaError_t launch_adam(float* params, const float* grad, float* m, float* v, int64_t n,
                        DeviceState* st, float lr, float beta1, float beta2, float eps,
                        int advance_it, cudaStream_t s) {
  k_adam<<<grid_for((n + 3) / 4), NT, 0, s>>>(params, grad, m, v, n, st, lr, beta1, beta2, eps);
  k_end_step<<<1, 1, 0, s>>>(st, advance_it);
  return cudaGetLastError();
}

cudaError_t launch_end_step(DeviceState* st, int advance_it, cudaStream_t s) {
  k_end_step<<<1, 1, 0, s>>>(st, advance_it);
  return cudaGetLastError();
}

cudaError_t launch_prolong(const float* src, float* dst, int64_t P, int N, int mode,
                           cudaStream_t s) {
  k_prolong<<<grid_for(2LL * N * P), NT, 0, s>>>(src, dst, P, N, mode);
  return cudaGetLastError();
}

cudaError_t launch_debug_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int64_t count,
                                uint32_t* out, cudaStream_t s) {
  k_debug_philox<<<(int)((count + NT - 1) / NT), NT, 0, s>>>(ctr, k0, k1, count, out);
  return cudaGetLastError();
}

cudaError_t launch_debug_dw(uint32_t it, int n, int64_t m0, int64_t count, int d, float sqrt_dt,
                            uint32_t k0, uint32_t k1, float* out, cudaStream_t s) {
  const int64_t th = count * ((d + 3) / 4);
  k_debug_dw<<<(int)((th + NT - 1) / NT), NT, 0, s>>>(it, n, m0, count, d, sqrt_dt, k0, k1, out);
  return cudaGetLastError();
}

}  // namespace bsde
