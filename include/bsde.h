/*
 * bsde.h — C-ABI of the B200-native deep-BSDE training hot path
 * (arXiv:1910.11623; BASELINE.json north_star).
 *
 * One call of bsde_train_step() is one training iteration of the per-step
 * Z-network scheme the paper describes at PAPER.md:78 (Han et al.: "there are N
 * different neural networks. Y0 and Z0 are treated as parameters and all the
 * Y_n are computed using an Euler discretization"), on the Euler-Maruyama
 * discretisation of Eq. 5:
 *
 *   ΔW_n ~ N(0, Δt)                       Eq. 5, PAPER.md:64   (Philox4x32-10, R8)
 *   X_{n+1} = X_n + √2 ΔW_n                Eq. 5; Eq. 12
 *   Z_n = W3 H2 + b3, H2 = H1 + ReLU(W2 H1 + b2), H1 = ReLU(W1 X_n + b1)
 *                                         Eq. 7, PAPER.md:217-219 (residual block, h = 1)
 *   Y_{n+1} = Y_n - f(Y_n, Z_n) Δt + Z_n·ΔW_n      Eq. 5, PAPER.md:66 with φ = -f (R2)
 *   L = (1/B) Σ_m (Y_N - g(X_N))²         Eq. 6, PAPER.md:75 (terminal term; R5)
 *   ∇L by a hand-written adjoint, summed over all ranks (NCCL), then Adam
 *                                         PAPER.md:319 (Adam), R6
 * and bsde_prolongate() is one level change of the multilevel schedule
 * (§3.2: h_l = h_0 M^-l, M = 2).
 * "R<k>" are the readings listed in DESIGN.md §Readings.
 *
 * Conventions for every call:
 *  - Return value: BSDE_OK (0) or a negative BSDE_E* code; never throws.
 *    bsde_last_error(ctx) returns a message naming the offending argument.
 *  - Host pointers are owned by the caller and only read/written during the call.
 *  - The library owns all device state of a context (parameters, gradients,
 *    Adam moments, scratch, the NCCL communicator) until bsde_destroy().
 *  - All device work is enqueued on cfg.stream.  Calls that return a host
 *    value computed on the device synchronise that stream.
 *  - A context is bound to one device and one rank and is not thread-safe.
 */
#ifndef BSDE_H_
#define BSDE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Problems (BASELINE.json configs; R10-R13). */
enum {
  BSDE_HEAT = 0,       /* f = 0,            g = |x|²            (config 1; R13)      */
  BSDE_HJB = 1,        /* f = -λ|z|²/2,     g = ln(0.5(1+|x|²))   */
  BSDE_ALLEN_CAHN = 2, /* f = y - y³,       g = 1/(2+0.4|x|²)   */
  BSDE_BLACK_SCHOLES = 3 /* X_{n+1} = X_n + σ X_n ⊙ ΔW_n, f = -r(y - Σz/σ), g = |x|²,
                            r = 0.05, σ = 0.4 (DESIGN R21)            */
};

/* GEMM operand precision; accumulation is always fp32 (R17, R18). */
enum {
  BSDE_FP32 = 0,       /* fp32-accurate: on tcgen05 ("tc32", kernel AUTO | TC) every GEMM
                          operand split into bf16 hi + lo and three MMAs per product
                          (hi·hi + hi·lo + lo·hi, ~2^-16 relative, DESIGN R18b); SIMT
                          FFMA with kernel SIMT, NAIS-Net or deterministic mode        */
  BSDE_BF16 = 1        /* bf16 operands, fp32 accumulate.  Per-step nets on tcgen05
                          (DESIGN R17): the biases are folded into the bf16 weight images,
                          H1 = bf16(ReLU(A1)), H2 = bf16(H1 + bf16(ReLU(A2))) (one bf16x2
                          add), ΔW_n enters the Y update's Z·ΔW and the adjoint's dZ as its
                          binary16 value; X, Y, the reductions and Adam are fp32         */
};

/* Kernel family selection. */
enum {
  BSDE_KERNEL_AUTO = 0,  /* tcgen05 when d+1 <= 128 and w+1 <= 128, else SIMT          */
  BSDE_KERNEL_SIMT = 1,  /* fp32 CUDA-core kernels (ignores precision: always fp32)    */
  BSDE_KERNEL_TC = 2     /* tcgen05 tensor-core kernels (sm_100a)                       */
};

/* a9: BSDE_PROLONG_COPY or BSDE_PROLONG_INTERP, optionally | BSDE_PROLONG_KEEP_ADAM
 * (R14b: the Adam moments m, v are prolonged by the same rule as the parameters and t
 * is kept, instead of the R14 reset; not with a sharded optimizer at world > 1) */
enum { BSDE_PROLONG_COPY = 0, BSDE_PROLONG_INTERP = 1, BSDE_PROLONG_KEEP_ADAM = 16 };

enum {
  BSDE_OK = 0,
  BSDE_EINVAL = -1,     /* bad argument; message names it                         */
  BSDE_ECUDA = -2,      /* CUDA runtime error (message has cudaGetErrorString)     */
  BSDE_ENCCL = -3,      /* NCCL error                                             */
  BSDE_EDIVERGED = -4,  /* loss non-finite or > 1e12, or non-finite gradient: the
                           Adam update of that step was skipped (SPEC S:425 reading) */
  BSDE_ESTATE = -5,     /* call not valid in the current state                    */
  BSDE_ENOMEM = -6      /* device allocation failed                               */
};

typedef struct bsde_ctx bsde_ctx;   /* opaque; one per GPU / rank */

typedef struct {
  int64_t batch_global;   /* B: paths per iteration summed over ranks; B % world == 0      */
  double x0;              /* X_0 = x0 * ones(d) (0 in configs 1-5; 0.1 for Black-Scholes) */
  double lambda;          /* HJB λ (1.0)                                                    */
  double lr, beta1, beta2, eps;  /* Adam (R6): per-config lr, 0.9, 0.999, 1e-8              */
  uint64_t seed;          /* Philox key = (seed mod 2^32, seed >> 32) (R8)                  */
  int precision;          /* BSDE_FP32 | BSDE_BF16                                          */
  int kernel;             /* BSDE_KERNEL_*                                                  */
  int prolong_mode;       /* BSDE_PROLONG_COPY | BSDE_PROLONG_INTERP, | BSDE_PROLONG_KEEP_ADAM */
  int max_levels;         /* buffers sized for N * 2^max_levels time steps                  */
  int device;             /* CUDA ordinal                                                   */
  void* stream;           /* cudaStream_t to enqueue on (NULL = legacy default stream)      */
  int rank, world;        /* this rank's index and the number of ranks (0, 1 for one GPU)  */
  const void* nccl_id;    /* 128-byte ncclUniqueId shared by all ranks (bsde_nccl_unique_id
                             on rank 0, broadcast by the caller): the context joins an NCCL
                             communicator of `world` ranks (world = 1 allowed).  NULL => no
                             collective: "fake-world" mode, the context computes its shard's
                             local gradient only (tests)                */
  int use_graph;          /* 1: capture the step in a CUDA graph and replay it              */
  int init_zero_head;     /* 1: W3 = 0 at init, so Z ≡ 0 (R7b; default for Allen-Cahn,
                             whose cubic driver diverges from a Xavier-initialised Z)      */
  int coupled_paths;      /* 1: coupled multilevel paths:
                             every level simulates the Brownian path of the finest grid
                             N_fine = N·2^max_levels; the increment of step n at the current
                             N is the sum of the f = N_fine/N fine increments it spans, each
                             drawn with Philox counter step n·f + j and √(T/N_fine) (R8).
                             0: each grid draws its own increments (default)               */
  int formulation;        /* BSDE_FORM_PER_STEP (default): N per-step Z-nets + trainable Y0,
                             terminal loss (BASELINE north_star).
                             BSDE_FORM_SHARED: the paper's own formulation (PAPER.md:69-77,
                             Eq. 6; DESIGN R23, R24): one network
                             u(t, x) of n_widths tanh layers shared by all steps, Y_n =
                             u(t_n, X_n), z_n = σ(X_n)ᵀ∇ₓu, residual-sum loss.  fp32 SIMT
                             GEMMs, or (precision BSDE_BF16, FC / ResNet) tcgen05 row and
                             weight-gradient GEMMs with bf16 operands                        */
  int sharded_adam;       /* 1 (with an NCCL communicator): reduce-scatter of the gradient,
                             Adam on this rank's 1/world shard of the parameters, all-gather
                             of the updated parameters (the optimizer half) in
                             place of the allreduce + replicated Adam.  Same arithmetic; after
                             bsde_train_step the gradient buffer holds the reduced values in
                             this rank's shard only (bsde_compute_grad still allreduces)    */
  int deterministic;      /* 1: fixed-order cross-CTA reductions (per-CTA partials of the
                             gradient, loss and dY0 summed in CTA order by one kernel) in
                             place of fp32/fp64 atomics, so repeated runs of the per-step
                             formulation are bitwise identical (SPEC determinism
                             invariant); the shared formulation rejects it (EINVAL)        */
  int shared_zN;          /* BSDE_FORM_SHARED: add the optional terminal term
                             Σ_m |∇ₓu(t_N, X_N) - ∇g(X_N)|² of PAPER.md:79 (DESIGN R27)    */
  void* workspace;        /* optional caller-owned device memory (e.g. a torch tensor) of
                             workspace_bytes >= bsde_workspace_bytes(): every device buffer
                             of the context is carved from it (256-byte aligned) and nothing
                             is cudaMalloc'ed; it must outlive the context.  NULL: the
                             library allocates and frees its own buffers                   */
  size_t workspace_bytes;
  int arch;               /* BSDE_FORM_SHARED: BSDE_ARCH_FC, BSDE_ARCH_RESNET (h_k = h_{k-1}
                             + tanh(W_k h_{k-1} + b_k) for k >= 2) or
                             BSDE_ARCH_NAIS (h_k = h_{k-1} + tanh(A_k h_{k-1} + B_k u + C_k),
                             A_k = -R_kᵀR_k - 0.01 I, u = (t, x); block layout [R_k C_k B_k
                             (w×(d+1))]; R_k projected after every Adam step; DESIGN R26).
                             BSDE_FORM_PER_STEP: BSDE_ARCH_NAIS replaces the residual block
                             by the NAIS-Net block H2 = H1 + ReLU(A H1 + B X_n + C), A =
                             -RᵀR - 0.01 I, with R projected onto ‖RᵀR‖_F <= 0.99 after every
                             Adam step (DESIGN R25); the
                             per-step layout becomes [W1 b1 R C W3 b3 B (w×d)]; fp32 SIMT
                             only.  Any other value: the R4 residual block              */
} bsde_config;

enum { BSDE_FORM_PER_STEP = 0, BSDE_FORM_SHARED = 1 };
enum { BSDE_ARCH_FC = 0, BSDE_ARCH_RESNET = 1, BSDE_ARCH_NAIS = 2 };

/* Fill *cfg with defaults: B = 256, x0 = 0, λ = 1, Adam (1e-2, 0.9, 0.999, 1e-8),
 * seed 0, FP32, KERNEL_AUTO, COPY, max_levels 0, device 0, default stream,
 * rank 0 of 1, no NCCL, graphs on, Xavier head (init_zero_head 0), uncoupled paths,
 * per-step formulation (FC arch for the shared one). */
void bsde_config_default(bsde_config* cfg);

/* Create a context for `problem` in dimension d with N time steps on [0, T]
 * (Δt = T/N, R16) and per-step Z-nets of hidden widths widths[0..n_widths)
 * (n_widths must be 2 with widths[0] == widths[1] = w: "d→w→w→d ReLU residual",
 * R4).  Parameters are initialised by R7 (Xavier-uniform weights, zero biases,
 * Y0 ~ U(0,1), from the Philox init stream keyed by cfg.seed), Adam state is zero
 * and the iteration counter is 0.  This rank owns global paths
 * [rank·B/world, (rank+1)·B/world).  Errors: EINVAL (shapes, B % world,
 * precision/kernel combination), ENOMEM, ECUDA, ENCCL. */
int bsde_create(int problem, int d, int N, double T, const int* widths, int n_widths,
                const bsde_config* cfg, bsde_ctx** out);

/* Device bytes a context with these arguments needs (the size of cfg.workspace
 * to pass to bsde_create); same validation and errors as bsde_create; nothing is
 * allocated, no stream or communicator is created (works without a GPU).  (T
 * does not change the size.) */
int bsde_workspace_bytes(int problem, int d, int N, const int* widths, int n_widths,
                         const bsde_config* cfg, size_t* bytes);

/* One training iteration: Philox ΔW for global
 * iteration `it`, forward rollout, terminal loss, adjoint, gradient allreduce
 * over the ranks, Adam.  Afterwards it += 1.  *loss_out (if non-NULL) receives the
 * loss of the parameters BEFORE the update (R20), mean over the global batch, and
 * the call synchronises; with loss_out == NULL the call is fully asynchronous.
 * Returns EDIVERGED (update skipped) if the loss is non-finite or > 1e12 or a
 * gradient is non-finite; with loss_out == NULL a divergence is reported by the
 * next synchronising call. */
int bsde_train_step(bsde_ctx* ctx, double* loss_out);

/* Multilevel level change (§3.2):
 * N <- 2N, Δt <- T/(2N); step k of the fine grid takes the coarse net k/2 (COPY)
 * or the midpoint rule (INTERP); Y0 is kept; Adam m, v, t are reset (R14), or with
 * BSDE_PROLONG_KEEP_ADAM m and v are prolonged by the same rule and t is kept (R14b);
 * the iteration counter continues.  `level` must equal the current level + 1 and be
 * <= cfg.max_levels.  Errors: ESTATE (also KEEP_ADAM with sharded_adam or the fused
 * optimizer at world > 1: each rank holds one shard of m, v). */
int bsde_prolongate(bsde_ctx* ctx, int level);

/* The trainable Y0 ≈ u(0, X0) (BASELINE.json north_star). Synchronises. */
int bsde_y0(const bsde_ctx* ctx, double* y0_out);

/* Introspection, checkpoint and resume.  The flat layout is
 * [Y0 | step 0: W1 (w×d) b1 (w) W2 (w×w) b2 (w) W3 (d×w) b3 (d) | step 1 | ...],
 * row-major fp32, 1 + N·(2dw + w² + 2w + d) values at the current N. */
int bsde_num_params(const bsde_ctx* ctx, int64_t* n);
int bsde_get_params(const bsde_ctx* ctx, float* host, int64_t n);
int bsde_set_params(bsde_ctx* ctx, const float* host, int64_t n);
/* Gradient of the last bsde_train_step / bsde_compute_grad (after the
 * allreduce), same layout. */
int bsde_get_grads(const bsde_ctx* ctx, float* host, int64_t n);
int bsde_get_adam_state(const bsde_ctx* ctx, float* m, float* v, int64_t n, int64_t* t);
int bsde_set_adam_state(bsde_ctx* ctx, const float* m, const float* v, int64_t n, int64_t t);
int bsde_get_iteration(const bsde_ctx* ctx, int64_t* it);
int bsde_set_iteration(bsde_ctx* ctx, int64_t it);     /* Philox counter position (R9) */
int bsde_current_steps(const bsde_ctx* ctx, int* N);

/* Forward + adjoint + allreduce of one iteration WITHOUT the Adam update and
 * without advancing the iteration counter (teacher-forced parity, R19).
 * *loss_out as in bsde_train_step.  Synchronises. */
int bsde_compute_grad(bsde_ctx* ctx, double* loss_out);

/* Forward-only loss on an evaluation stream: Philox counter word 3 is
 * 0x80000000 | eval_id, global paths [0, batch) of which this rank takes its
 * share; summed over ranks.  Synchronises. */
int bsde_eval_loss(bsde_ctx* ctx, uint32_t eval_id, int64_t batch, double* loss_out);

/* Test hooks for bit-parity of the generator (SURVEY.md pin H0): the raw
 * Philox4x32-10 outputs for `count` counters ctr[4*i..4*i+3] under key
 * (key[0], key[1]), and the increments ΔW_n for global paths
 * [m0, m0+count) at iteration it (host out[count×d], fp32).  Both run on the
 * device with the same code the training kernels use.  Synchronise. */
int bsde_debug_philox(const bsde_ctx* ctx, const uint32_t* ctr, const uint32_t key[2],
                      int64_t count, uint32_t* out);
int bsde_debug_dw(const bsde_ctx* ctx, int64_t it, int n, int64_t m0, int64_t count,
                  float* host_out);
/* As bsde_debug_dw, with the MUFU-based Box-Muller the tcgen05 kernels use
 * (same counter and map, R8; |error| ~ 1e-6 relative to the exact map). */
int bsde_debug_dw_fast(const bsde_ctx* ctx, int64_t it, int n, int64_t m0, int64_t count,
                       float* host_out);
/* Terminal residuals R^m = Y_N^m - g(X_N^m) of the last training forward pass
 * for this rank's local paths [m0, m0+count) (global path rank·B/world + m):
 * sampled full-size parity (R19).  host_out[count] fp32.  Synchronises. */
int bsde_debug_residuals(const bsde_ctx* ctx, int64_t m0, int64_t count, float* host_out);

/* Test hook for the tcgen05 operand layouts: one
 * M=128, N=112 bf16 UMMA on the current device with fp32 host inputs rounded to
 * bf16.  mode 0: D[128×112] = A[128×112]·B[112×112]ᵀ (both K-major);
 * mode 1: D = A[128×112]·B[112×112] (B MN-major); mode 2: D = A[128×112]ᵀ·B[128×112]
 * (both MN-major, rows >= 112 of D undefined); mode 3: as mode 0 with A staged in
 * tensor memory (the forward's TMEM A operands).  Row-major host arrays.  Synchronises. */
int bsde_debug_umma(int mode, const float* a, const float* b, float* d_out);

/* Profiling hook: runs one forward (which = 0) or forward + adjoint (which = 1)
 * pass of the current iteration with a clock64() trace of CTA 0 enabled and
 * copies up to n stamps to host out[] (16 slots per step/item, 0 = unused; see
 * tc.cu CLK points; all zero unless the library was built with
 * -DBSDE_PHASE_CLOCKS).  Overwrites the gradient buffer.  tcgen05 path only.
 * Synchronises. */
int bsde_debug_phase_clocks(bsde_ctx* ctx, int which, uint64_t* out, int n);

/* Profiling hook for the bench's roofline figures: runs `steps` training
 * iterations (eagerly, no graph) with CUDA events recorded on cfg.stream
 * between the phases of the step and returns the mean duration of each phase
 * in milliseconds: ms_out[0] begin (zero grad), [1] forward kernel, [2] adjoint
 * kernel, [3] allreduce, [4] check, [5] Adam (+ bf16 weight pack).
 * n_out must be >= 6.  Synchronises. */
int bsde_profile_steps(bsde_ctx* ctx, int steps, float* ms_out, int n_out);

/* NEXT-4 (BASELINE north_star (e)): the gradient
 * reduce-scatter, Adam on this rank's 1/world shard of the parameters and the
 * all-gather of the updated parameters as ONE kernel over peer memory (NVLink loads /
 * stores through CUDA IPC mappings, fused_opt.cu), chained after the adjoint in the
 * step graph in place of the NCCL allreduce + check + Adam.  Shards are reduced in
 * rank order (deterministic); the divergence guard is decided over all ranks.
 *   bsde_ipc_export writes 4 cudaIpcMemHandle_t (256 bytes: gradient, parameters,
 *     barrier flags, device state) to out[bytes >= 256].  Not with cfg.workspace.
 *   bsde_fused_opt_enable takes every rank's 256 bytes in rank order (world × 256;
 *     NULL allowed at world = 1), opens the peers' buffers and switches
 *     bsde_train_step to the fused kernel.  Every rank must enable it; all ranks
 *     then run the same number of steps (the kernel's barriers span the ranks).
 * One block per SM must be co-resident (nothing else on the GPU while it runs).
 * Collective over the ranks; EINVAL on a world mismatch, ESTATE if already enabled. */
int bsde_ipc_export(const bsde_ctx* ctx, void* out, int64_t bytes);
int bsde_fused_opt_enable(bsde_ctx* ctx, const void* handles, int world);

/* Number of kernels the last bsde_train_step enqueued (for the bench's
 * gpu_launches), and the name of the kernel family in use ("simt" | "tc" bf16 |
 * "tc32" fp32-accurate bf16x3 row GEMMs | "shared-simt" | "shared-tc"). */
int bsde_launches_per_step(const bsde_ctx* ctx, int* n);
const char* bsde_kernel_family(const bsde_ctx* ctx);

/* NCCL unique id for bsde_config.nccl_id (call on rank 0; 128 bytes). */
int bsde_nccl_unique_id(void* out128);

/* Message of the last error on ctx (ctx may be NULL: last create error on this thread). */
const char* bsde_last_error(const bsde_ctx* ctx);

void bsde_destroy(bsde_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* BSDE_H_ */
