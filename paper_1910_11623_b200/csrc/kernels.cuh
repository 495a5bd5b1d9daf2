// kernels.cuh — argument blocks and launchers of every device kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace bsde {

// Arguments of one forward/adjoint pass.  Everything a graph replay needs to
// change from step to step lives in DeviceState (it, t), not here.
struct PassArgs {
  int problem, d, w, N;
  float dt, sqrt_dt, lam, x0, inv_B;   // Δt, √Δt, λ, X0 component, 1/B_global
  int64_t B_local, m0;                 // this rank's paths: global [m0, m0 + B_local)
  uint32_t k0, k1;                     // Philox key (R8)
  int eval;                            // 1: forward only, counter word 3 = eval_it
  uint32_t eval_it;
  const float* params;                 // fp32 master (flat layout)
  float* grad;                         // flat gradient (+ nothing else); zeroed per step
  float* Xstore;                       // [N][B_local][d] fp32: X_n for the adjoint pass
  // ā recursion ā_n = ā_{n+1} f_n, f_n = 1 - Δt ∂_y f(Y_n), in product form: the
  // forward stores the prefix products P_{n+1} = f_0 ⋯ f_n and ā_N P_N, so that
  // ā_{n+1} = ā_N P_N / P_{n+1} needs no backward scan (per_step_abar problems)
  float* Pstore;                       // [N][B_local]: P_{n+1} (per_step_abar problems only)
  float* abar;                         // [B_local]: ā_N P_N (per_step_abar) or ā_N
  float* Rstore;                       // [B_local] terminal residual R (debug / parity)
  DeviceState* state;
  double* loss_acc;                    // Σ_m R² accumulator (state->loss_sum or eval slot)
  // tcgen05 path only
  const void* wpack;                   // packed bf16 weight images (see tc.cu)
  void* xpack;                         // bf16 X store (BF16 precision)
  float* gpart;                        // SIMT adjoint: per-CTA scratch gradients
  void* dwpack;                        // tcgen05 path: fp16 ΔW_n images (written by k_fwd_tc)
  unsigned long long* clk;             // debug: per-phase clock64() trace of CTA 0 (or null)
  int precision;
  int nais;                            // NAIS-Net block in the per-step nets (R25)
  // deterministic mode (cfg.deterministic): the kernels write per-CTA partials in
  // place of cross-CTA atomics and k_det_reduce sums them in a fixed order
  float* dpart;                        // [grid][dseg][P_step] adjoint gradient partials
  int dseg;                            // step segments per adjoint CTA
  double* lpart;                       // [forward grid] Σ R² partials
  float* y0part;                       // [forward grid] dY0 partials
  int cpl;                             // coupled paths: fine steps per step (1 = uncoupled)
  float sqrt_dt_f;                     // √(Δt/cpl)
};

// NEXT-4 (fused_opt.cu): reduce-scatter + sharded Adam + all-gather over peer memory
constexpr int kMaxPeers = 8;
struct FusedOptArgs {
  int world, rank;
  int64_t np, shard;                       // parameters (unpadded), shard (multiple of 4)
  float* peer_grad[kMaxPeers];             // every rank's gradient buffer (IPC-mapped; [rank] = own)
  float* peer_params[kMaxPeers];
  unsigned* peer_flags[kMaxPeers];         // [0] arrivals, [1+q] divergence of rank q, [16] grid barrier
  DeviceState* peer_state[kMaxPeers];
  float *m, *v;                            // this rank's Adam moments (shard entries used)
  DeviceState* state;
  double inv_B;
  float lr, beta1, beta2, eps;
};
cudaError_t launch_fused_opt(const FusedOptArgs& a, int sms, cudaStream_t s);

// fp32-accurate per-step nets on tcgen05 (rows_tc.cu; DESIGN R18b): one iteration's
// row buffers over R = N·B rows (row (n, m) = n·B + m), bf16x3 GEMM operands
struct RowsArgs {
  int problem, d, w, N, Dp, Wp;        // Dp = pad16(d+1), Wp = pad16(w+1)
  float dt, sqrt_dt_f, lam, x0, inv_B;
  int cpl;                             // coupled paths: fine steps per step
  int64_t B, m0;                       // local paths (rows per step), first global path
  int64_t Bs;                          // row stride per step of the [N][Bs][·] row buffers: B, or
                                       // B rounded up to 128-row tiles for the tile-image formats
  uint32_t k0, k1;
  int eval;
  uint32_t eval_it;
  DeviceState* state;
  double* loss_acc;
  const float* params;
  float* grad;
  const uint8_t* wimg;                 // per step: W̃1, W̃2, W̃3 bf16 hi images, then lo images
  uint8_t* wimg_w;                     // the same, for the pack kernel
  float *XT, *GW, *H1, *H2, *DH, *DA;  // X̃ [R×Dp]; ΔW then G = ΔW - Δt∂_z f [R×Dp]; H1, H2, dH2, dA1 [R×Wp]
  float *S, *xn2;                      // per row (Z·ΔW, |Z|² | Σ Z); |X_N|² per path
  // ReLU masks per row (compile-time shapes): 1[A1 > 0], 1[A2 > 0] as 4 words, bit l of
  // word e = column 4l + e (written by F1 / F2, read by the fused adjoint B12)
  uint32_t *M1, *M2;
  float *abar, *Pstore, *Rstore;       // as PassArgs
};
bool rows_supported(int d, int w);
size_t rows_buffer_bytes(int d, int w, int N, int64_t B);
size_t rows_pack_bytes(int d, int w, int N);
void rows_carve(RowsArgs& a, void* base, int N_max);
cudaError_t launch_rows_pack(const RowsArgs& a, cudaStream_t s);
cudaError_t launch_rows_forward(const RowsArgs& a, cudaStream_t s, int* launches);
cudaError_t launch_rows_backward(const RowsArgs& a, cudaStream_t s, int* launches);

// Shared-network formulation (shared.cu): one
// iteration's device state.  Rows r = n·M + m, n = 0..N, row-major buffers.
constexpr int kMaxSharedLayers = 8;
struct ShArgs {
  int problem, arch, d, w, L, N, K0p;       // K0p = d+1 rounded up to 4 (row stride of U0, G0, Ḡ0)
  int64_t M, m0;                            // local paths, first global path
  float dt, sqrt_dt_f, lam, x0, inv_B;
  int cpl;                                  // coupled paths: fine steps per step (R22)
  uint32_t k0, k1;
  int eval;
  uint32_t eval_it;
  DeviceState* state;
  double* loss_acc;
  const float* params;
  float* grad;
  float* Rstore;                            // [M] terminal residuals r_N
  int64_t off_W[kMaxSharedLayers], off_v;   // flat offsets of W_k (b_k follows) and v (c follows)
  int64_t off_Bk[kMaxSharedLayers];         // NAIS-Net (arch 2): B_k of block k ≥ 1 (R26)
  float* Am;                                // NAIS-Net: A_k = -R_kᵀR_k - εI, [L][w×w]
  int tc;                                   // 1: bf16 tcgen05 row GEMMs (cfg.precision BF16)
  int zN;                                   // the optional Σ|∇ₓu(t_N, X_N) - ∇g(X_N)|² term (R27)
  uint16_t* wimg;                           // tc: bf16 UMMA images of W_k [w × pad16(K_in)]
  int64_t off_img[kMaxSharedLayers];        // tc: element offset of layer k's image
  float *U0, *G0, *G0b, *dW;                // [R×K0p] inputs, ∇u, ∂L/∂∇u;  [N·M×d] increments
  float* S[kMaxSharedLayers];               // s_k = tanh(a_k)
  float* H[kMaxSharedLayers];               // h_k (= S[k] unless residual)
  float* D[kMaxSharedLayers];               // δ_k = g_k ⊙ (1 - s_k²)
  float* G[kMaxSharedLayers];               // g_k = ∂u/∂h_k, k < L-1 (g_{L-1} = v)
  float* Sb[kMaxSharedLayers];              // s̄_k from the input-gradient adjoint
  float* HL;
  float *Gb[2], *Ab[2], *Hb[2];             // ping-pong ḡ, ā, h̄
  float *u, *ub, *q;                        // [R] u, ū; [R×4] z·ΔW | |z|² | Σz
};
size_t shared_num_params(int d, int w, int L, int arch);
void shared_offsets(ShArgs& a);
size_t shared_buffer_bytes(int d, int w, int L, int arch, int N_max, int64_t M);
void shared_carve(ShArgs& a, void* base, int N_max);
cudaError_t launch_shared_init(float* params, const ShArgs& a, uint32_t k0, uint32_t k1,
                               cudaStream_t s);
cudaError_t launch_shared_point(const ShArgs& a, float* out, cudaStream_t s);
cudaError_t launch_shared_nais_project(const ShArgs& a, float* params, cudaStream_t s);
cudaError_t launch_shared_step(const ShArgs& a, cudaStream_t s, cudaEvent_t mid, int* launches);

// deterministic reduction of the partials (aux.cu): grad[step n] = Σ_c dpart[c][n - n_first(c)]
// over the adjoint CTAs c covering step n in ascending order, grad[0] = Σ_c y0part[c],
// *loss_acc = Σ_c lpart[c] (fixed order); bwd_grid = 0 for a forward-only (eval) pass
cudaError_t launch_det_reduce(const PassArgs& a, int fwd_grid, int bwd_grid, int64_t items,
                              int ntiles, cudaStream_t s);
int det_segments(int64_t items, int grid, int ntiles);

// SIMT fp32 kernels (simt.cu)
cudaError_t launch_fwd_simt(const PassArgs& a, cudaStream_t s);
cudaError_t launch_bwd_simt(const PassArgs& a, cudaStream_t s);

// auxiliary kernels (aux.cu)
cudaError_t launch_init_params(float* params, int d, int w, int N, uint32_t k0, uint32_t k1,
                               int zero_head, int nais, cudaStream_t s);
// NAIS-Net (R25): R_n ← R_n((1-ε)/‖RᵀR‖_F)^½ where ‖RᵀR‖_F > 1-ε, every step n;
// and the gradient transform Ā -> R̄ = -R(Ā + Āᵀ) in the W2 slot of each step
cudaError_t launch_nais_project(float* params, int d, int w, int N, cudaStream_t s);
cudaError_t launch_nais_grad(const float* params, float* grad, int d, int w, int N, cudaStream_t s);
cudaError_t launch_begin_step(DeviceState* st, float* grad, int64_t n_grad, cudaStream_t s);
cudaError_t launch_check(const float* grad, int64_t n, DeviceState* st, double inv_B,
                         float beta1, float beta2, cudaStream_t s);
cudaError_t launch_adam(float* params, const float* grad, float* m, float* v, int64_t n,
                        DeviceState* st, float lr, float beta1, float beta2, float eps,
                        int advance_it, cudaStream_t s);
cudaError_t launch_end_step(DeviceState* st, int advance_it, cudaStream_t s);
cudaError_t launch_prolong(const float* src, float* dst, int64_t P, int N, int mode,
                           cudaStream_t s);
cudaError_t launch_debug_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int64_t count,
                                uint32_t* out, cudaStream_t s);
cudaError_t launch_debug_dw(uint32_t it, int n, int64_t m0, int64_t count, int d,
                            float sqrt_dt, uint32_t k0, uint32_t k1, float* out,
                            cudaStream_t s);

}  // namespace bsde
