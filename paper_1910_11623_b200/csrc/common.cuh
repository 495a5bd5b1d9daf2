// common.cuh — device building blocks shared by the SIMT and tcgen05 kernels.
//
//  * Philox4x32-10 (Salmon et al., SC'11) and the Box-Muller map that turn a
//    counter (q, m, n, it) into 4 standard normals: Eq. 5
//    "ΔW_n ~ N(0, Δt_n)"; reading R8 in DESIGN.md.
//  * The three problems' driver f and terminal g: PAPER.md:300-313, readings
//    R2, R10-R13 (Han sign convention Y_{n+1} = Y_n - f Δt + Z·ΔW).
//  * The flat parameter layout of include/bsde.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bsde {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;
constexpr uint32_t kEvalBit = 0x80000000u;     // counter word 3 of evaluation streams
constexpr uint32_t kInitStream = 0xC0000000u;  // counter word 3 of the init stream (R7)

enum { kHeat = 0, kHJB = 1, kAllenCahn = 2, kBlackScholes = 3 };
constexpr float kNaisEps = 0.01f;   // A = -RᵀR - εI ("ε = 0.01 in our case"); h = 1
// Black-Scholes constants ("d = 100, r = 0.05 and σ = 0.4")
constexpr float kBSRate = 0.05f, kBSSigma = 0.4f;

// 10 rounds; the key is warp-uniform, so ptxas folds the key schedule into
// immediates / uniform registers and each round is 2 IMAD.WIDE + 2 LOP3.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += kPhiloxW0; k1 += kPhiloxW1; }
    const uint32_t lo0 = kPhiloxM0 * c.x, hi0 = __umulhi(kPhiloxM0, c.x);
    const uint32_t lo1 = kPhiloxM1 * c.z, hi1 = __umulhi(kPhiloxM1, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// u = ((x >> 9) + 0.5) 2^-23 ∈ (0,1): exact in fp32 (R8).
__device__ __forceinline__ float unit_from_u32(uint32_t x) {
  return (__uint2float_rn(x >> 9) + 0.5f) * 1.1920928955078125e-07f;
}

// Box-Muller with IEEE-accurate logf/sqrtf/sincospif (no fast-math on this path):
// z0 = r cos(2πu2), z1 = r sin(2πu2), r = sqrt(-2 ln u1).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& z0, float& z1) {
  const float u1 = unit_from_u32(a), u2 = unit_from_u32(b);
  const float r = sqrtf(-2.0f * logf(u1));
  float s, c;
  sincospif(2.0f * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// Normals 4q..4q+3 of (path m, step n, iteration it): ctr = (q, m, n, it).
__device__ __forceinline__ float4 normals4(uint32_t q, uint32_t m, uint32_t n, uint32_t it,
                                           uint32_t k0, uint32_t k1) {
  const uint4 x = philox4x32_10(make_uint4(q, m, n, it), k0, k1);
  float4 z;
  box_muller(x.x, x.y, z.x, z.y);
  box_muller(x.z, x.w, z.z, z.w);
  return z;
}

// ---- fast Box-Muller for the tensor-core kernels (same map as R8) ----------
// u = ((x >> 9) + 1/2) 2^-23 via the exponent trick (exact): 1.m - (1 - 2^-24).
__device__ __forceinline__ float unit_fast(uint32_t x) {
  return __int_as_float((int)((x >> 9) | 0x3F800000u)) - 0.99999994039535522f;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// √Δt·(r cos 2πu2, r sin 2πu2), r = sqrt(-2 ln u1), with MUFU lg2 / sqrt / sin / cos.
// ln u1 for u1 > 1 - 2^-6 uses the series of log1p(-v), v = 1 - u1 (exact), so
// the relative accuracy of r holds near u1 = 1 where lg2.approx's absolute
// error would dominate.  The angle is reduced to (-π, π): 2πu2 - π, so
// cos(2πu2) = -cos(a), sin(2πu2) = -sin(a).  Typical |error| ~ 1e-6 (pinned by
// tests/test_gpu_tc.py::test_fast_normals_match_oracle).
__device__ __forceinline__ void box_muller_fast(uint32_t xa, uint32_t xb, float sdt, float& z0,
                                                float& z1) {
  const uint32_t k = xa >> 9;
  const float u1 = unit_fast(xa);
  // -2 ln(u1): series of -2 log1p(-v), v = 1 - u1 (exact: Sterbenz) for u1 > 1 - 2^-6,
  // else -2 ln2 · lg2.approx(u1); both evaluated, selected without a branch.
  const float v = 1.0f - u1;
  const float r2s = v * fmaf(v, fmaf(v, fmaf(v, 0.5f, 0.66666667f), 1.0f), 2.0f);
  float l2;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(u1));
  const float r2 = k >= 0x7E0000u ? r2s : -1.38629436111989061f * l2;
  const float r = sqrt_approx(r2) * sdt;
  // angle 2π(u2 - 1/2) ∈ (-π, π); u2 - 1/2 by the same exponent trick (exact)
  const float a = (__int_as_float((int)((xb >> 9) | 0x3F800000u)) - 1.49999994039535522f) *
                  6.28318530717958648f;
  float s, c;
  __sincosf(a, &s, &c);
  z0 = -r * c;
  z1 = -r * s;
}

// √Δt · normals 4q..4q+3 of (m, n, it): the increments ΔW of R8, fast map.
__device__ __forceinline__ float4 dw4_fast(uint32_t q, uint32_t m, uint32_t n, uint32_t it,
                                           uint32_t k0, uint32_t k1, float sdt) {
  const uint4 x = philox4x32_10(make_uint4(q, m, n, it), k0, k1);
  float4 z;
  box_muller_fast(x.x, x.y, sdt, z.x, z.y);
  box_muller_fast(x.z, x.w, sdt, z.z, z.w);
  return z;
}

// ---- problems (R2, R10-R13, R21) -------------------------------------------
// f(y, z) given |z|² and Σ z_i; ∂f/∂y; ∂f/∂z = c·z + c0·1 (the scalars c, c0);
// g(s = |x|²); the Euler step of X (μ = 0).
__device__ __forceinline__ float driver_f(int problem, float y, float zz, float sz, float lam) {
  if (problem == kHJB) return -0.5f * lam * zz;
  if (problem == kAllenCahn) return y - y * y * y;
  if (problem == kBlackScholes) return -kBSRate * (y - sz * (1.0f / kBSSigma));
  return 0.0f;
}
__device__ __forceinline__ float driver_dfdy(int problem, float y) {
  if (problem == kAllenCahn) return 1.0f - 3.0f * y * y;
  if (problem == kBlackScholes) return -kBSRate;
  return 0.0f;
}
__device__ __forceinline__ float driver_dfdz_coef(int problem, float lam) {
  return problem == kHJB ? -lam : 0.0f;
}
__device__ __forceinline__ float driver_dfdz_const(int problem) {
  return problem == kBlackScholes ? kBSRate / kBSSigma : 0.0f;
}
// ā_n = ā_{n+1}(1 - Δt ∂_y f) varies with n: the adjoint reads a per-step ā
__host__ __device__ __forceinline__ bool per_step_abar(int problem) {
  return problem == kAllenCahn || problem == kBlackScholes;
}
__device__ __forceinline__ float terminal_g(int problem, float s) {
  if (problem == kHJB) return logf(0.5f * (1.0f + s));
  if (problem == kAllenCahn) return 1.0f / (2.0f + 0.4f * s);
  return s;   // heat, Black-Scholes: |x|²
}
// X_{n+1} = X_n + σ ΔW_n with σ = √2 I, or σ X_n ⊙ ΔW_n (Black-Scholes)
__device__ __forceinline__ float x_step(int problem, float x, float dw) {
  return problem == kBlackScholes ? fmaf(kBSSigma * dw, x, x) : fmaf(1.41421356237309515f, dw, x);
}

// ---- flat parameter layout (include/bsde.h) -------------------------------
struct NetDims {
  int d, w;
  int nais = 0;   // NAIS-Net block (R25): W2/b2 slots hold R/C and B (w×d) follows b3
  __host__ __device__ int64_t step_size() const {
    return 2LL * d * w + 1LL * w * w + 2LL * w + d + (nais ? 1LL * w * d : 0LL);
  }
  __host__ __device__ int64_t off_W1() const { return 0; }
  __host__ __device__ int64_t off_b1() const { return 1LL * w * d; }
  __host__ __device__ int64_t off_W2() const { return off_b1() + w; }
  __host__ __device__ int64_t off_b2() const { return off_W2() + 1LL * w * w; }
  __host__ __device__ int64_t off_W3() const { return off_b2() + w; }
  __host__ __device__ int64_t off_b3() const { return off_W3() + 1LL * d * w; }
  __host__ __device__ int64_t off_B() const { return off_b3() + d; }
  // parameters of step n start at 1 + n * step_size() (index 0 is Y0)
  __host__ __device__ int64_t step_base(int n) const { return 1 + (int64_t)n * step_size(); }
};

// Per-context device scalars, advanced on the device so that a captured CUDA
// graph of the step replays correctly.
struct DeviceState {
  uint32_t it;        // global iteration = Philox counter word 3 (R9)
  int32_t t;          // Adam step count (t of the last update)
  int32_t diverged;   // set by the check kernel for the current step (sticky copy below)
  int32_t diverged_any;
  double loss_sum;    // Σ_m R² of the current step (local, then all-reduced)
  double loss_last;   // loss of the last step (mean over the global batch)
  float c1, c2;       // Adam bias corrections 1/(1-β1^(t+1)), 1/(1-β2^(t+1)) of this step
  uint32_t opt_epoch; // launches of the fused peer-memory optimizer (fused_opt.cu)
};

}  // namespace bsde
