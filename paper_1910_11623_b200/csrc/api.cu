// api.cu — the C-ABI of include/bsde.h: context lifetime, validation, the
// per-iteration launch sequence (optionally captured in a CUDA graph), the NCCL
// gradient allreduce (a7, loaded with dlopen so the library has no link-time
// NCCL dependency), multilevel prolongation and the introspection calls.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (SURVEY §5 tracing)

#include "bsde.h"
#include "kernels.cuh"

namespace bsde {
size_t simt_max_smem(int d, int w);
bool simt_supported(int d, int w);
size_t simt_pack_bytes(int d, int w, int N, int nais);
size_t simt_xstore_bytes(int d, int N, int64_t B_local);
size_t simt_scratch_bytes(int d, int w, int nais);
cudaError_t launch_pack_simt(const PassArgs& a, cudaStream_t s);
bool tc_supported(int d, int w);
cudaError_t launch_fwd_tc(const PassArgs& a, cudaStream_t s);
cudaError_t launch_bwd_tc(const PassArgs& a, cudaStream_t s);
cudaError_t launch_pack_weights(const PassArgs& a, cudaStream_t s);
size_t tc_pack_bytes(int d, int w, int N, int precision);
size_t tc_xstore_bytes(int d, int w, int N, int64_t B_local);
cudaError_t launch_umma_test(int mode, const float* A, const float* B, float* D, cudaStream_t s);
cudaError_t launch_debug_dw_fast(uint32_t it, int n, int64_t m0, int64_t count, int d,
                                 float sqrt_dt, uint32_t k0, uint32_t k1, float* out,
                                 cudaStream_t s);
}  // namespace bsde

using namespace bsde;

namespace {

thread_local std::string g_create_error;
thread_local size_t* g_dry_run = nullptr;   // set by bsde_workspace_bytes around bsde_create

// ---- NCCL, resolved at run time --------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
    a.ReduceScatter = (decltype(a.ReduceScatter))dlsym(h, "ncclReduceScatter");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.GroupStart &&
           a.ReduceScatter && a.AllGather &&
           a.GroupEnd && a.GetErrorString;
    return a;
  }();
  return api;
}

}  // namespace

struct bsde_ctx {
  int problem = 0, d = 0, w = 0, N = 0, N0 = 0, level = 0, N_max = 0;
  bool shared = false;          // BSDE_FORM_SHARED (NEXT-1)
  int nais = 0;                 // per-step nets with the NAIS-Net block (NEXT-2, R25)
  int L = 0;                    // shared: number of tanh layers
  void* shbuf = nullptr;        // shared: row buffers (carved into ShArgs)
  void* rowsbuf = nullptr;      // fp32-accurate tcgen05 family: row buffers (RowsArgs)
  unsigned* flags = nullptr;    // NEXT-4 fused optimizer: barrier counters / divergence flags
  bool fused = false;           // bsde_fused_opt_enable done: the peer-memory optimizer runs
  FusedOptArgs fo{};            // its peer pointers (np / shard filled per step)
  std::vector<void*> ipc_open;  // peer mappings to close
  bool external_ws = false;     // buffers carved from cfg.workspace (caller-owned)
  int sms = 148;                // SM count (grid sizes of the deterministic partials)
  float* dpart = nullptr;       // deterministic mode: adjoint partials
  double* lpart = nullptr;      // deterministic mode: forward loss partials [256]
  float* y0part = nullptr;      // deterministic mode: forward dY0 partials [256]
  double T = 1.0;
  bsde_config cfg{};
  int64_t B_local = 0, m0 = 0;
  int family = BSDE_KERNEL_SIMT;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  float *params = nullptr, *grad = nullptr, *adam_m = nullptr, *adam_v = nullptr;
  float *scratch = nullptr, *Xstore = nullptr, *Pstore = nullptr, *abar = nullptr;
  float* Rstore = nullptr;
  void* wpack = nullptr;
  void* xpack = nullptr;        // tcgen05 path: fp16 ΔW_n images
  float* gpart = nullptr;
  DeviceState* state = nullptr;
  double* eval_loss = nullptr;
  ncclComm_t comm = nullptr;
  cudaGraphExec_t graph = nullptr;
  int graph_N = -1;
  int launches = 0;
  int64_t host_it = 0;   // mirror of state->it
  std::string err;
};

namespace {

int fail(bsde_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf; else g_create_error = buf;
  return code;
}

#define CK(expr)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(ctx, BSDE_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),     \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define NK(expr)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return fail(ctx, BSDE_ENCCL, "%s: %s", #expr, nccl().GetErrorString(r_));         \
  } while (0)

// sharded Adam (NEXT-4): parameters and gradient padded to world × shard floats, shard % 4 == 0
int64_t shard_of(const bsde_ctx* c, int64_t np) {
  const int64_t per = (np + c->cfg.world - 1) / c->cfg.world;
  return (per + 3) / 4 * 4;
}

// launch geometry of the per-step kernels (tc.cu / simt.cu launchers): tiles of
// 128 (tcgen05) or 64 (SIMT) paths, forward grid min(tiles, SMs), adjoint grid
// min(N·tiles, SMs)
void det_geometry(const bsde_ctx* c, int N, int* fwd_grid, int* bwd_grid, int* ntiles,
                  int64_t* items) {
  const int tile = c->family == BSDE_KERNEL_TC ? 128 : 64;
  *ntiles = (int)((c->B_local + tile - 1) / tile);
  *items = (int64_t)N * *ntiles;
  *fwd_grid = *ntiles < c->sms ? *ntiles : c->sms;
  *bwd_grid = (int)(*items < c->sms ? *items : c->sms);
}

int64_t num_params_at(const bsde_ctx* c, int N) {
  if (c->shared) return (int64_t)shared_num_params(c->d, c->w, c->L, c->cfg.arch);   // independent of N
  return 1 + (int64_t)N * NetDims{c->d, c->w, c->nais}.step_size();
}

ShArgs sh_args(bsde_ctx* c) {
  ShArgs a{};
  a.problem = c->problem;
  a.arch = c->cfg.arch;
  a.d = c->d;
  a.w = c->w;
  a.L = c->L;
  a.N = c->N;
  a.K0p = (c->d + 1 + 3) & ~3;
  a.M = c->B_local;
  a.m0 = c->m0;
  a.dt = (float)(c->T / c->N);
  a.cpl = c->cfg.coupled_paths ? c->N_max / c->N : 1;
  a.sqrt_dt_f = (float)std::sqrt(c->T / ((double)c->N * a.cpl));
  a.lam = (float)c->cfg.lambda;
  a.x0 = (float)c->cfg.x0;
  a.inv_B = (float)(1.0 / (double)c->cfg.batch_global);
  a.k0 = (uint32_t)(c->cfg.seed & 0xffffffffu);
  a.k1 = (uint32_t)(c->cfg.seed >> 32);
  a.state = c->state;
  a.loss_acc = &c->state->loss_sum;
  a.params = c->params;
  a.grad = c->grad;
  a.Rstore = c->Rstore;
  a.tc = c->cfg.precision == BSDE_BF16 ? 1 : 0;
  a.zN = c->cfg.shared_zN;
  shared_offsets(a);
  if (c->shbuf) shared_carve(a, c->shbuf, c->N_max);
  return a;
}

// internal kernel family: the per-step nets at BSDE_FP32 on tcgen05 (bf16x3 row GEMMs,
// rows_tc.cu); the public kernel enum asks for it as BSDE_KERNEL_TC with BSDE_FP32
constexpr int kFamilyRows = 3;

RowsArgs rows_args(bsde_ctx* c, int64_t B, int64_t m0) {
  RowsArgs a{};
  a.problem = c->problem;
  a.d = c->d;
  a.w = c->w;
  a.N = c->N;
  a.dt = (float)(c->T / c->N);
  a.cpl = c->cfg.coupled_paths ? c->N_max / c->N : 1;
  a.sqrt_dt_f = (float)std::sqrt(c->T / ((double)c->N * a.cpl));
  a.lam = (float)c->cfg.lambda;
  a.x0 = (float)c->cfg.x0;
  a.inv_B = (float)(1.0 / (double)c->cfg.batch_global);
  a.B = B;
  a.m0 = m0;
  a.k0 = (uint32_t)(c->cfg.seed & 0xffffffffu);
  a.k1 = (uint32_t)(c->cfg.seed >> 32);
  a.state = c->state;
  a.loss_acc = &c->state->loss_sum;
  a.params = c->params;
  a.grad = c->grad;
  a.wimg = static_cast<const uint8_t*>(c->wpack);
  a.wimg_w = static_cast<uint8_t*>(c->wpack);
  a.abar = c->abar;
  a.Pstore = c->Pstore;
  a.Rstore = c->Rstore;
  rows_carve(a, c->rowsbuf, c->N_max);
  return a;
}

PassArgs pass_args(bsde_ctx* c) {
  PassArgs a{};
  a.problem = c->problem;
  a.d = c->d;
  a.w = c->w;
  a.N = c->N;
  a.dt = (float)(c->T / c->N);
  a.sqrt_dt = (float)std::sqrt(c->T / c->N);
  a.cpl = c->cfg.coupled_paths ? c->N_max / c->N : 1;
  a.sqrt_dt_f = (float)std::sqrt(c->T / ((double)c->N * a.cpl));
  a.lam = (float)c->cfg.lambda;
  a.x0 = (float)c->cfg.x0;
  a.inv_B = (float)(1.0 / (double)c->cfg.batch_global);
  a.B_local = c->B_local;
  a.m0 = c->m0;
  a.k0 = (uint32_t)(c->cfg.seed & 0xffffffffu);
  a.k1 = (uint32_t)(c->cfg.seed >> 32);
  a.params = c->params;
  a.grad = c->grad;
  a.Xstore = c->Xstore;
  a.Pstore = c->Pstore;
  a.abar = c->abar;
  a.Rstore = c->Rstore;
  a.state = c->state;
  a.loss_acc = &c->state->loss_sum;
  a.wpack = c->wpack;
  a.xpack = c->Xstore;   // the tcgen05 path stores X_n as bf16 operand images
  a.gpart = c->gpart;
  a.dwpack = c->xpack;
  a.precision = c->cfg.precision;
  a.nais = c->nais;
  if (c->cfg.deterministic) {
    a.dpart = c->dpart;
    a.lpart = c->lpart;
    a.y0part = c->y0part;
    int fg, bg, nt;
    int64_t items;
    det_geometry(c, c->N, &fg, &bg, &nt, &items);
    a.dseg = det_segments(items, bg, nt);
  }
  return a;
}

// Enqueue one iteration; with_update = 0 stops after the gradient + check.
// ev (optional, 7 events) brackets the phases for bsde_profile_steps.
int enqueue_step(bsde_ctx* ctx, bool with_update, cudaEvent_t* ev = nullptr) {
  const int64_t np = num_params_at(ctx, ctx->N);
  const PassArgs a = pass_args(ctx);
  // phase events (bsde_profile_steps) and NVTX ranges named after the §8(a) rows;
  // the ranges mark the enqueue (capture) of each phase for nsys timelines
  static const char* const kPhase[6] = {"bsde.begin", "bsde.fwd (a1-a5)", "bsde.adjoint (a6)",
                                        "bsde.allreduce (a7)", "bsde.check", "bsde.adam (a8)"};
  int open_range = -1;
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], ctx->stream);
    if (open_range >= 0) nvtxRangePop();
    open_range = i < 6 ? i : -1;
    if (open_range >= 0) nvtxRangePushA(kPhase[i]);
  };
  int launches = 0;
  mark(0);
  const bool sharded = ctx->comm && ctx->cfg.sharded_adam && with_update;
  const int64_t shard = shard_of(ctx, np), npad = shard * ctx->cfg.world;
  CK(launch_begin_step(ctx->state, ctx->grad, (sharded || ctx->fused) ? npad : np, ctx->stream));
  launches += 1;   // k_begin_step (the memset is not a kernel)
  mark(1);
  if (ctx->shared) {
    int nl = 0;
    CK(launch_shared_step(sh_args(ctx), ctx->stream, ev ? ev[2] : nullptr, &nl));
    launches += nl;
  } else if (ctx->family == kFamilyRows) {
    const RowsArgs ra = rows_args(ctx, ctx->B_local, ctx->m0);
    CK(launch_rows_forward(ra, ctx->stream, &launches));
    mark(2);
    CK(launch_rows_backward(ra, ctx->stream, &launches));
  } else if (ctx->family == BSDE_KERNEL_TC) {
    CK(launch_fwd_tc(a, ctx->stream));
    mark(2);
    CK(launch_bwd_tc(a, ctx->stream));
    launches += 2;
    if (ctx->cfg.deterministic) {
      int fg, bg, nt;
      int64_t items;
      det_geometry(ctx, ctx->N, &fg, &bg, &nt, &items);
      CK(launch_det_reduce(a, fg, bg, items, nt, ctx->stream));
      launches += 1;
    }
  } else {
    CK(launch_fwd_simt(a, ctx->stream));
    mark(2);
    CK(launch_bwd_simt(a, ctx->stream));
    launches += 2;
    if (ctx->cfg.deterministic) {
      int fg, bg, nt;
      int64_t items;
      det_geometry(ctx, ctx->N, &fg, &bg, &nt, &items);
      CK(launch_det_reduce(a, fg, bg, items, nt, ctx->stream));
      launches += 1;
    }
    if (ctx->nais) {   // Ā (W2 slot) -> R̄ = -R(Ā + Āᵀ), R25
      CK(launch_nais_grad(ctx->params, ctx->grad, ctx->d, ctx->w, ctx->N, ctx->stream));
      launches += 1;
    }
  }
  mark(3);
  if (ctx->fused && with_update) {   // NEXT-4: one peer-memory kernel replaces a7 + check + a8
    FusedOptArgs fo = ctx->fo;
    fo.np = np;
    fo.shard = shard;
    fo.inv_B = 1.0 / (double)ctx->cfg.batch_global;
    CK(launch_fused_opt(fo, ctx->sms, ctx->stream));
    mark(4);
    mark(5);
    CK(launch_end_step(ctx->state, 1, ctx->stream));
    launches += 2;
    if (ctx->nais) {
      CK(launch_nais_project(ctx->params, ctx->d, ctx->w, ctx->N, ctx->stream));
      launches += 1;
    }
    if (!ctx->shared) {
      if (ctx->family == kFamilyRows) CK(launch_rows_pack(rows_args(ctx, ctx->B_local, ctx->m0), ctx->stream));
      else if (ctx->family == BSDE_KERNEL_TC) CK(launch_pack_weights(a, ctx->stream));
      else CK(launch_pack_simt(a, ctx->stream));
      launches += 1;
    }
    mark(6);
    ctx->launches = launches;
    return BSDE_OK;
  }
  const int64_t off = sharded ? shard * ctx->cfg.rank : 0;
  const int64_t nloc = sharded ? std::max<int64_t>(0, std::min(shard, np - off)) : np;
  if (sharded) {   // reduce-scatter: this rank's shard of the summed gradient, in place
    NK(nccl().GroupStart());
    NK(nccl().ReduceScatter(ctx->grad, ctx->grad + off, (size_t)shard, ncclFloat32, ncclSum,
                            ctx->comm, ctx->stream));
    NK(nccl().AllReduce(&ctx->state->loss_sum, &ctx->state->loss_sum, 1, ncclFloat64, ncclSum,
                        ctx->comm, ctx->stream));
    NK(nccl().GroupEnd());
  } else if (ctx->comm) {
    NK(nccl().GroupStart());
    NK(nccl().AllReduce(ctx->grad, ctx->grad, (size_t)np, ncclFloat32, ncclSum, ctx->comm,
                        ctx->stream));
    NK(nccl().AllReduce(&ctx->state->loss_sum, &ctx->state->loss_sum, 1, ncclFloat64, ncclSum,
                        ctx->comm, ctx->stream));
    NK(nccl().GroupEnd());
  }
  mark(4);
  CK(launch_check(ctx->grad + off, nloc, ctx->state, 1.0 / (double)ctx->cfg.batch_global,
                  (float)ctx->cfg.beta1, (float)ctx->cfg.beta2, ctx->stream));
  launches += 1;
  if (sharded)   // a non-finite gradient in any shard skips the update on every rank
    NK(nccl().AllReduce(&ctx->state->diverged, &ctx->state->diverged, 1, ncclInt32, ncclMax,
                        ctx->comm, ctx->stream));
  mark(5);
  if (with_update) {
    CK(launch_adam(ctx->params + off, ctx->grad + off, ctx->adam_m + off, ctx->adam_v + off, nloc,
                   ctx->state, (float)ctx->cfg.lr, (float)ctx->cfg.beta1, (float)ctx->cfg.beta2,
                   (float)ctx->cfg.eps, 1, ctx->stream));
    launches += 2;
    if (sharded)   // every rank gets the updated parameters of every shard
      NK(nccl().AllGather(ctx->params + off, ctx->params, (size_t)shard, ncclFloat32, ctx->comm,
                          ctx->stream));
    if (ctx->nais) {   // projection of every R_n after the optimizer step (R25)
      CK(launch_nais_project(ctx->params, ctx->d, ctx->w, ctx->N, ctx->stream));
      launches += 1;
    }
    if (ctx->shared && ctx->cfg.arch == BSDE_ARCH_NAIS) {   // every block's R_k (R26)
      CK(launch_shared_nais_project(sh_args(ctx), ctx->params, ctx->stream));
      launches += 1;
    }
    // weight images for the next step (bf16 UMMA images / fp32 transposed images)
    if (!ctx->shared) {
      if (ctx->family == kFamilyRows) CK(launch_rows_pack(rows_args(ctx, ctx->B_local, ctx->m0), ctx->stream));
      else if (ctx->family == BSDE_KERNEL_TC) CK(launch_pack_weights(a, ctx->stream));
      else CK(launch_pack_simt(a, ctx->stream));
      launches += 1;
    }
  }
  mark(6);
  ctx->launches = launches;
  return BSDE_OK;
}

int read_state(bsde_ctx* ctx, DeviceState* hs) {
  CK(cudaMemcpyAsync(hs, ctx->state, sizeof(DeviceState), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}

int repack(bsde_ctx* ctx) {
  if (ctx->shared) return BSDE_OK;   // the shared kernels read the fp32 master directly
  if (ctx->family == kFamilyRows) CK(launch_rows_pack(rows_args(ctx, ctx->B_local, ctx->m0), ctx->stream));
  else if (ctx->family == BSDE_KERNEL_TC) CK(launch_pack_weights(pass_args(ctx), ctx->stream));
  else CK(launch_pack_simt(pass_args(ctx), ctx->stream));
  return BSDE_OK;
}

void free_all(bsde_ctx* c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
  c->ipc_open.clear();
  if (c->external_ws) {   // nothing of ours to free but the communicator and the stream
    if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    return;
  }
  void* bufs[] = {c->params, c->grad, c->adam_m, c->adam_v, c->scratch, c->Xstore, c->Pstore,
                  c->abar, c->Rstore, c->wpack, c->xpack, c->gpart, c->state,
                  c->eval_loss, c->shbuf, c->dpart, c->lpart, c->y0part, c->rowsbuf, c->flags};
  for (void* p : bufs)
    if (p) cudaFree(p);
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
}

}  // namespace

extern "C" {

void bsde_config_default(bsde_config* cfg) {
  std::memset(cfg, 0, sizeof *cfg);
  cfg->batch_global = 256;
  cfg->x0 = 0.0;
  cfg->lambda = 1.0;
  cfg->lr = 1e-2;
  cfg->beta1 = 0.9;
  cfg->beta2 = 0.999;
  cfg->eps = 1e-8;
  cfg->seed = 0;
  cfg->precision = BSDE_FP32;
  cfg->kernel = BSDE_KERNEL_AUTO;
  cfg->prolong_mode = BSDE_PROLONG_COPY;
  cfg->max_levels = 0;
  cfg->device = 0;
  cfg->stream = nullptr;
  cfg->rank = 0;
  cfg->world = 1;
  cfg->nccl_id = nullptr;
  cfg->use_graph = 1;
  cfg->init_zero_head = 0;
}

int bsde_nccl_unique_id(void* out128) {
  bsde_ctx* ctx = nullptr;
  if (!out128) return fail(ctx, BSDE_EINVAL, "out128 is NULL");
  if (!nccl().ok) return fail(ctx, BSDE_ENCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NK(nccl().GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
  return BSDE_OK;
}

int bsde_create(int problem, int d, int N, double T, const int* widths, int n_widths,
                const bsde_config* cfg_in, bsde_ctx** out) {
  bsde_ctx* none = nullptr;
  if (!out) return fail(none, BSDE_EINVAL, "out is NULL");
  *out = nullptr;
  bsde_config cfg;
  if (cfg_in) cfg = *cfg_in; else bsde_config_default(&cfg);
  if (problem < BSDE_HEAT || problem > BSDE_BLACK_SCHOLES)
    return fail(none, BSDE_EINVAL, "problem=%d not in {0 heat, 1 hjb, 2 allen_cahn, 3 black_scholes}",
                problem);
  if (d < 1 || N < 1 || !(T > 0.0))
    return fail(none, BSDE_EINVAL, "need d >= 1, N >= 1, T > 0 (got d=%d N=%d T=%g)", d, N, T);
  const bool shared = cfg.formulation == BSDE_FORM_SHARED;
  if (cfg.formulation != BSDE_FORM_PER_STEP && !shared)
    return fail(none, BSDE_EINVAL, "formulation=%d", cfg.formulation);
  if (shared) {
    if (!widths || n_widths < 1 || n_widths > kMaxSharedLayers || widths[0] < 1)
      return fail(none, BSDE_EINVAL, "shared net: 1 <= n_widths <= %d layers of width w >= 1",
                  kMaxSharedLayers);
    for (int k = 1; k < n_widths; ++k)
      if (widths[k] != widths[0])
        return fail(none, BSDE_EINVAL, "shared net: all layer widths must be equal (R23)");
    if (cfg.arch != BSDE_ARCH_FC && cfg.arch != BSDE_ARCH_RESNET && cfg.arch != BSDE_ARCH_NAIS)
      return fail(none, BSDE_EINVAL, "arch=%d", cfg.arch);
    if (cfg.precision == BSDE_BF16 && cfg.arch == BSDE_ARCH_NAIS)
      return fail(none, BSDE_EINVAL, "the shared NAIS-Net network runs on the fp32 kernels only");
    if (cfg.deterministic)
      return fail(none, BSDE_EINVAL, "deterministic mode covers the per-step formulation only");
    if (widths[0] % 4)   // the activation rows (stride w) are read as float4 by the GEMMs
      return fail(none, BSDE_EINVAL, "shared net: width w=%d must be a multiple of 4", widths[0]);
  } else if (!widths || n_widths != 2 || widths[0] != widths[1] || widths[0] < 1) {
    return fail(none, BSDE_EINVAL,
                "widths must be {w, w} with w >= 1 (d->w->w->d residual net, R4); got n_widths=%d",
                n_widths);
  }
  const int w = widths[0];
  if (cfg.world < 1 || cfg.rank < 0 || cfg.rank >= cfg.world)
    return fail(none, BSDE_EINVAL, "rank=%d world=%d", cfg.rank, cfg.world);
  if (cfg.batch_global < 1 || cfg.batch_global % cfg.world != 0)
    return fail(none, BSDE_EINVAL, "batch_global=%lld must be >= 1 and divisible by world=%d",
                (long long)cfg.batch_global, cfg.world);
  if (cfg.batch_global > (int64_t)1 << 32)
    return fail(none, BSDE_EINVAL, "batch_global=%lld exceeds 2^32 (Philox path word)",
                (long long)cfg.batch_global);
  if (cfg.precision != BSDE_FP32 && cfg.precision != BSDE_BF16)
    return fail(none, BSDE_EINVAL, "precision=%d", cfg.precision);
  if (cfg.max_levels < 0 || cfg.max_levels > 12)
    return fail(none, BSDE_EINVAL, "max_levels=%d", cfg.max_levels);
  if ((cfg.prolong_mode & ~BSDE_PROLONG_KEEP_ADAM) != BSDE_PROLONG_COPY &&
      (cfg.prolong_mode & ~BSDE_PROLONG_KEEP_ADAM) != BSDE_PROLONG_INTERP)
    return fail(none, BSDE_EINVAL, "prolong_mode=%d", cfg.prolong_mode);
  if (!(cfg.lr > 0) || !(cfg.beta1 >= 0 && cfg.beta1 < 1) || !(cfg.beta2 >= 0 && cfg.beta2 < 1) ||
      !(cfg.eps > 0))
    return fail(none, BSDE_EINVAL, "Adam hyper-parameters out of range");
  const int nais = (!shared && cfg.arch == BSDE_ARCH_NAIS) ? 1 : 0;
  if (nais && (cfg.precision != BSDE_FP32 || cfg.kernel == BSDE_KERNEL_TC))
    return fail(none, BSDE_EINVAL, "the NAIS-Net block runs on the fp32 SIMT kernels only (R25)");
  int family = cfg.kernel;
  if (shared || nais) family = BSDE_KERNEL_SIMT;
  // fp32-accurate precision on tcgen05: bf16x3 row GEMMs (R18b); the fixed-order
  // reductions of deterministic mode exist on the SIMT kernels only
  const bool rows_ok = !shared && !nais && rows_supported(d, w) && !cfg.deterministic;
  if (family == BSDE_KERNEL_AUTO)
    family = (cfg.precision == BSDE_BF16 && tc_supported(d, w)) ? BSDE_KERNEL_TC
             : (cfg.precision == BSDE_FP32 && rows_ok)          ? kFamilyRows
                                                                : BSDE_KERNEL_SIMT;
  if (family == BSDE_KERNEL_TC && cfg.precision == BSDE_FP32) {
    if (!rows_ok)
      return fail(none, BSDE_EINVAL,
                  "fp32 on tcgen05 needs d+1, w+1 <= 128, the residual block and deterministic=0 "
                  "(got d=%d w=%d); use kernel=SIMT", d, w);
    family = kFamilyRows;
  }
  if (family == BSDE_KERNEL_TC && !tc_supported(d, w))
    return fail(none, BSDE_EINVAL,
                "no tcgen05 instantiation for d=%d w=%d (built: 100/110, 10/20, 37/45; d+1, w+1 <= 128)",
                d, w);
  if (family == BSDE_KERNEL_SIMT && cfg.precision == BSDE_BF16 && !shared)
    return fail(none, BSDE_EINVAL, "bf16 operands need the tcgen05 kernels (kernel=SIMT given)");
  if (family == BSDE_KERNEL_SIMT && !shared && !simt_supported(d, w))
    return fail(none, BSDE_EINVAL, "d=%d w=%d too large for the SIMT kernels (d, w <= 127 and shared "
                "memory)", d, w);
  if (family != BSDE_KERNEL_SIMT && family != BSDE_KERNEL_TC && family != kFamilyRows)
    return fail(none, BSDE_EINVAL, "kernel=%d", cfg.kernel);
  if (cfg.nccl_id && !nccl().ok)
    return fail(none, BSDE_ENCCL, "nccl_id given (world=%d) but libnccl.so.2 could not be loaded",
                cfg.world);

  bsde_ctx* ctx = new bsde_ctx;
  ctx->problem = problem;
  ctx->shared = shared;
  ctx->nais = nais;
  ctx->L = shared ? n_widths : 0;
  ctx->d = d;
  ctx->w = w;
  ctx->N = ctx->N0 = N;
  ctx->N_max = N << cfg.max_levels;
  ctx->T = T;
  ctx->cfg = cfg;
  ctx->family = family;
  ctx->B_local = cfg.batch_global / cfg.world;
  ctx->m0 = (int64_t)cfg.rank * ctx->B_local;

  auto bail = [&](int code) {
    g_create_error = ctx->err;
    free_all(ctx);
    delete ctx;
    return code;
  };
  {
    int dev = cfg.device, nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
      ctx->sms = nsm;
    else
      cudaGetLastError();   // no device (bsde_workspace_bytes on a CPU box): keep 148
  }
  size_t det_floats = 0;   // deterministic mode: max over the levels of grid × segments × P_step
  if (cfg.deterministic && !shared) {
    const int64_t P = NetDims{d, w, nais}.step_size();
    for (int l = 0, Nl = N; l <= cfg.max_levels; ++l, Nl *= 2) {
      int fg, bg, nt;
      int64_t items;
      det_geometry(ctx, Nl, &fg, &bg, &nt, &items);
      det_floats = std::max(det_floats, (size_t)bg * det_segments(items, bg, nt) * P);
    }
  }
  const int64_t npmax = num_params_at(ctx, ctx->N_max);
  const int64_t npalloc = std::max<int64_t>(npmax, shard_of(ctx, npmax) * cfg.world);   // NEXT-4 padding
  struct Alloc { void** p; size_t bytes; };
  // X_n store for the adjoint: fp32 rows (SIMT) or bf16 operand images (tcgen05)
  const size_t xs = (shared || family == kFamilyRows) ? 16
                   : family == BSDE_KERNEL_TC ? tc_xstore_bytes(d, w, ctx->N_max, ctx->B_local)
                                              : simt_xstore_bytes(d, ctx->N_max, ctx->B_local);
  std::vector<Alloc> allocs = {
      {(void**)&ctx->params, npalloc * sizeof(float)},
      {(void**)&ctx->grad, npalloc * sizeof(float)},
      {(void**)&ctx->adam_m, npalloc * sizeof(float)},
      {(void**)&ctx->adam_v, npalloc * sizeof(float)},
      {(void**)&ctx->scratch, npmax * sizeof(float)},
      {(void**)&ctx->Xstore, xs},
      {(void**)&ctx->abar, (size_t)ctx->B_local * sizeof(float)},
      {(void**)&ctx->Rstore, (size_t)ctx->B_local * sizeof(float)},
      {(void**)&ctx->state, sizeof(DeviceState)},
      {(void**)&ctx->eval_loss, sizeof(double) * 2},
      {(void**)&ctx->flags, 32 * sizeof(unsigned)},
  };
  if (det_floats) {
    allocs.push_back({(void**)&ctx->dpart, det_floats * sizeof(float)});
    allocs.push_back({(void**)&ctx->lpart, 256 * sizeof(double)});
    allocs.push_back({(void**)&ctx->y0part, 256 * sizeof(float)});
  }
  if (shared) {
    allocs.push_back({&ctx->shbuf, shared_buffer_bytes(d, w, ctx->L, cfg.arch, ctx->N_max,
                                                       ctx->B_local)});
  } else if (per_step_abar(problem)) {
    allocs.push_back({(void**)&ctx->Pstore, (size_t)ctx->N_max * ctx->B_local * sizeof(float)});
  }
  if (shared) {
  } else if (family == kFamilyRows) {
    allocs.push_back({&ctx->wpack, rows_pack_bytes(d, w, ctx->N_max)});
    allocs.push_back({&ctx->rowsbuf, rows_buffer_bytes(d, w, ctx->N_max, ctx->B_local)});
  } else if (family == BSDE_KERNEL_TC) {
    allocs.push_back({&ctx->wpack, tc_pack_bytes(d, w, ctx->N_max, cfg.precision)});
    allocs.push_back({&ctx->xpack, tc_xstore_bytes(d, w, ctx->N_max, ctx->B_local)});
  } else {
    allocs.push_back({&ctx->wpack, simt_pack_bytes(d, w, ctx->N_max, nais)});
    allocs.push_back({(void**)&ctx->gpart, simt_scratch_bytes(d, w, nais)});
  }
  size_t ws_total = 0;
  for (auto& al : allocs) ws_total += (al.bytes + 255) / 256 * 256;
  if (g_dry_run) {   // bsde_workspace_bytes
    *g_dry_run = ws_total;
    delete ctx;
    return BSDE_OK;
  }
  {
    cudaError_t e = cudaSetDevice(cfg.device);
    if (e != cudaSuccess) { ctx->err = std::string("cudaSetDevice: ") + cudaGetErrorString(e); return bail(BSDE_ECUDA); }
  }
  if (cfg.stream) {
    ctx->stream = (cudaStream_t)cfg.stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      ctx->err = "cudaStreamCreate failed";
      return bail(BSDE_ECUDA);
    }
    ctx->own_stream = true;
  }
  if (cfg.workspace) {   // carve every buffer from the caller's memory
    if (cfg.workspace_bytes < ws_total || ((uintptr_t)cfg.workspace & 255u)) {
      ctx->err = "workspace too small or not 256-byte aligned (need " + std::to_string(ws_total) +
                 " bytes)";
      return bail(BSDE_EINVAL);
    }
    uint8_t* base = static_cast<uint8_t*>(cfg.workspace);
    for (auto& al : allocs) {
      *al.p = base;
      base += (al.bytes + 255) / 256 * 256;
    }
    ctx->external_ws = true;
  } else {
    for (auto& al : allocs) {
      cudaError_t e = cudaMalloc(al.p, al.bytes);
      if (e != cudaSuccess) {
        char b[256];
        snprintf(b, sizeof b, "cudaMalloc(%zu bytes): %s", al.bytes, cudaGetErrorString(e));
        ctx->err = b;
        return bail(BSDE_ENOMEM);
      }
    }
  }
  cudaMemsetAsync(ctx->adam_m, 0, npalloc * sizeof(float), ctx->stream);
  cudaMemsetAsync(ctx->adam_v, 0, npalloc * sizeof(float), ctx->stream);
  cudaMemsetAsync(ctx->params, 0, npalloc * sizeof(float), ctx->stream);
  cudaMemsetAsync(ctx->state, 0, sizeof(DeviceState), ctx->stream);
  cudaMemsetAsync(ctx->flags, 0, 32 * sizeof(unsigned), ctx->stream);
  const cudaError_t ie =
      shared ? launch_shared_init(ctx->params, sh_args(ctx), (uint32_t)(cfg.seed & 0xffffffffu),
                                  (uint32_t)(cfg.seed >> 32), ctx->stream)
             : launch_init_params(ctx->params, d, w, N, (uint32_t)(cfg.seed & 0xffffffffu),
                                  (uint32_t)(cfg.seed >> 32), cfg.init_zero_head, nais, ctx->stream);
  if (ie != cudaSuccess) {
    ctx->err = "init kernel launch failed";
    return bail(BSDE_ECUDA);
  }
  if (repack(ctx) != BSDE_OK) return bail(BSDE_ECUDA);
  if (cfg.nccl_id) {   // any world size, including a 1-rank communicator
    ncclUniqueId id;
    std::memcpy(&id, cfg.nccl_id, sizeof id);
    ncclResult_t r = nccl().CommInitRank(&ctx->comm, cfg.world, id, cfg.rank);
    if (r != ncclSuccess) {
      ctx->err = std::string("ncclCommInitRank: ") + nccl().GetErrorString(r);
      ctx->comm = nullptr;
      return bail(BSDE_ENCCL);
    }
  }
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    ctx->err = std::string("create: ") + cudaGetErrorString(cudaGetLastError());
    return bail(BSDE_ECUDA);
  }
  *out = ctx;
  return BSDE_OK;
}

int bsde_workspace_bytes(int problem, int d, int N, const int* widths, int n_widths,
                         const bsde_config* cfg, size_t* bytes) {
  if (!bytes) return fail(nullptr, BSDE_EINVAL, "bytes is NULL");
  bsde_ctx* none = nullptr;
  g_dry_run = bytes;
  const int rc = bsde_create(problem, d, N, 1.0, widths, n_widths, cfg, &none);
  g_dry_run = nullptr;
  return rc;
}

int bsde_train_step(bsde_ctx* ctx, double* loss_out) {
  if (!ctx) return fail(ctx, BSDE_EINVAL, "ctx is NULL");
  if (ctx->cfg.use_graph) {
    if (!ctx->graph || ctx->graph_N != ctx->N) {
      if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_step(ctx, true);
      cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
      if (rc != BSDE_OK) { if (e == cudaSuccess) cudaGraphDestroy(g); return rc; }
      CK(e);
      cudaError_t ie = cudaGraphInstantiate(&ctx->graph, g, 0);
      cudaGraphDestroy(g);
      CK(ie);
      ctx->graph_N = ctx->N;
    }
    CK(cudaGraphLaunch(ctx->graph, ctx->stream));
  } else {
    int rc = enqueue_step(ctx, true);
    if (rc != BSDE_OK) return rc;
  }
  ctx->host_it += 1;
  if (loss_out) {
    DeviceState hs;
    int rc = read_state(ctx, &hs);
    if (rc != BSDE_OK) return rc;
    *loss_out = hs.loss_last;
    if (hs.diverged_any) return fail(ctx, BSDE_EDIVERGED,
                                     "diverged: loss=%g (non-finite or > 1e12, or non-finite gradient); update skipped",
                                     hs.loss_last);
  }
  return BSDE_OK;
}

int bsde_compute_grad(bsde_ctx* ctx, double* loss_out) {
  if (!ctx) return fail(ctx, BSDE_EINVAL, "ctx is NULL");
  int rc = enqueue_step(ctx, false);
  if (rc != BSDE_OK) return rc;
  DeviceState hs;
  rc = read_state(ctx, &hs);
  if (rc != BSDE_OK) return rc;
  if (loss_out) *loss_out = hs.loss_last;
  return BSDE_OK;
}

int bsde_prolongate(bsde_ctx* ctx, int level) {
  if (!ctx) return fail(ctx, BSDE_EINVAL, "ctx is NULL");
  if (level != ctx->level + 1 || level > ctx->cfg.max_levels)
    return fail(ctx, BSDE_ESTATE, "prolongate(level=%d): current level %d, max_levels %d", level,
                ctx->level, ctx->cfg.max_levels);
  const int pmode = ctx->cfg.prolong_mode & ~BSDE_PROLONG_KEEP_ADAM;
  const bool keep = (ctx->cfg.prolong_mode & BSDE_PROLONG_KEEP_ADAM) != 0;   // R14b
  if (keep && ctx->cfg.world > 1 && (ctx->cfg.sharded_adam || ctx->fused))
    return fail(ctx, BSDE_ESTATE, "prolongate: KEEP_ADAM with a sharded optimizer (each rank "
                                  "holds one shard of the Adam moments)");
  if (!ctx->shared) {   // the shared network is the same function on every grid
    const int64_t P = NetDims{ctx->d, ctx->w, ctx->nais}.step_size();
    const int64_t np = num_params_at(ctx, ctx->N);
    float* bufs[3] = {ctx->params, ctx->adam_m, ctx->adam_v};
    for (int b = 0; b < (keep ? 3 : 1); ++b) {   // parameters, then (R14b) m and v by the same rule
      CK(cudaMemcpyAsync(ctx->scratch, bufs[b], np * sizeof(float), cudaMemcpyDeviceToDevice,
                         ctx->stream));
      CK(launch_prolong(ctx->scratch, bufs[b], P, ctx->N, pmode, ctx->stream));
    }
  }
  ctx->N *= 2;
  ctx->level = level;
  const int64_t np2 = num_params_at(ctx, ctx->N);
  int rc;
  if (!keep) {   // R14: the optimizer restarts on the fine grid
    CK(cudaMemsetAsync(ctx->adam_m, 0, np2 * sizeof(float), ctx->stream));
    CK(cudaMemsetAsync(ctx->adam_v, 0, np2 * sizeof(float), ctx->stream));
    DeviceState hs;
    rc = read_state(ctx, &hs);
    if (rc != BSDE_OK) return rc;
    hs.t = 0;
    CK(cudaMemcpyAsync(ctx->state, &hs, sizeof hs, cudaMemcpyHostToDevice, ctx->stream));
  }
  rc = repack(ctx);
  if (rc != BSDE_OK) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}

int bsde_y0(const bsde_ctx* cctx, double* y0_out) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(cctx);
  if (!ctx || !y0_out) return fail(ctx, BSDE_EINVAL, "NULL argument");
  float y;
  if (ctx->shared) {   // Y0 = u(0, X_0), evaluated by the network on the device
    CK(launch_shared_point(sh_args(ctx), ctx->scratch, ctx->stream));
    CK(cudaMemcpyAsync(&y, ctx->scratch, sizeof y, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    CK(cudaMemcpyAsync(&y, ctx->params, sizeof y, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  *y0_out = y;
  return BSDE_OK;
}

int bsde_num_params(const bsde_ctx* ctx, int64_t* n) {
  if (!ctx || !n) return fail(const_cast<bsde_ctx*>(ctx), BSDE_EINVAL, "NULL argument");
  *n = num_params_at(ctx, ctx->N);
  return BSDE_OK;
}

static int copy_out(bsde_ctx* ctx, const float* dev, float* host, int64_t n) {
  if (!host || n != num_params_at(ctx, ctx->N))
    return fail(ctx, BSDE_EINVAL, "buffer of %lld floats given, %lld expected", (long long)n,
                (long long)num_params_at(ctx, ctx->N));
  CK(cudaMemcpyAsync(host, dev, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}

static int copy_in(bsde_ctx* ctx, float* dev, const float* host, int64_t n) {
  if (!host || n != num_params_at(ctx, ctx->N))
    return fail(ctx, BSDE_EINVAL, "buffer of %lld floats given, %lld expected", (long long)n,
                (long long)num_params_at(ctx, ctx->N));
  CK(cudaMemcpyAsync(dev, host, n * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}

int bsde_get_params(const bsde_ctx* c, float* host, int64_t n) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(c);
  if (!ctx) return BSDE_EINVAL;
  return copy_out(ctx, ctx->params, host, n);
}
int bsde_set_params(bsde_ctx* ctx, const float* host, int64_t n) {
  if (!ctx) return BSDE_EINVAL;
  int rc = copy_in(ctx, ctx->params, host, n);
  if (rc != BSDE_OK) return rc;
  rc = repack(ctx);
  if (rc != BSDE_OK) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}
int bsde_get_grads(const bsde_ctx* c, float* host, int64_t n) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(c);
  if (!ctx) return BSDE_EINVAL;
  return copy_out(ctx, ctx->grad, host, n);
}
int bsde_get_adam_state(const bsde_ctx* c, float* m, float* v, int64_t n, int64_t* t) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(c);
  if (!ctx || !t) return BSDE_EINVAL;
  int rc = copy_out(ctx, ctx->adam_m, m, n);
  if (rc == BSDE_OK) rc = copy_out(ctx, ctx->adam_v, v, n);
  if (rc != BSDE_OK) return rc;
  DeviceState hs;
  rc = read_state(ctx, &hs);
  *t = hs.t;
  return rc;
}
int bsde_set_adam_state(bsde_ctx* ctx, const float* m, const float* v, int64_t n, int64_t t) {
  if (!ctx || t < 0) return BSDE_EINVAL;
  int rc = copy_in(ctx, ctx->adam_m, m, n);
  if (rc == BSDE_OK) rc = copy_in(ctx, ctx->adam_v, v, n);
  if (rc != BSDE_OK) return rc;
  DeviceState hs;
  rc = read_state(ctx, &hs);
  if (rc != BSDE_OK) return rc;
  hs.t = (int32_t)t;
  CK(cudaMemcpyAsync(ctx->state, &hs, sizeof hs, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}
int bsde_get_iteration(const bsde_ctx* c, int64_t* it) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(c);
  if (!ctx || !it) return BSDE_EINVAL;
  DeviceState hs;
  int rc = read_state(ctx, &hs);
  *it = hs.it;
  return rc;
}
int bsde_set_iteration(bsde_ctx* ctx, int64_t it) {
  if (!ctx || it < 0 || it >= (int64_t)kEvalBit)
    return fail(ctx, BSDE_EINVAL, "iteration must be in [0, 2^31)");
  DeviceState hs;
  int rc = read_state(ctx, &hs);
  if (rc != BSDE_OK) return rc;
  hs.it = (uint32_t)it;
  hs.diverged_any = 0;
  CK(cudaMemcpyAsync(ctx->state, &hs, sizeof hs, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->host_it = it;
  return BSDE_OK;
}
int bsde_current_steps(const bsde_ctx* ctx, int* N) {
  if (!ctx || !N) return BSDE_EINVAL;
  *N = ctx->N;
  return BSDE_OK;
}

int bsde_eval_loss(bsde_ctx* ctx, uint32_t eval_id, int64_t batch, double* loss_out) {
  if (!ctx || !loss_out) return fail(ctx, BSDE_EINVAL, "NULL argument");
  if (batch < 1 || batch % ctx->cfg.world || batch > ((int64_t)1 << 32))
    return fail(ctx, BSDE_EINVAL, "eval batch=%lld must be divisible by world=%d",
                (long long)batch, ctx->cfg.world);
  if (ctx->shared) {   // the rank's eval paths in chunks of at most B_local rows per step
    const int64_t per_rank = batch / ctx->cfg.world, first = (int64_t)ctx->cfg.rank * per_rank;
    CK(cudaMemsetAsync(ctx->eval_loss, 0, sizeof(double), ctx->stream));
    for (int64_t c0 = 0; c0 < per_rank; c0 += ctx->B_local) {
      ShArgs sa = sh_args(ctx);
      sa.eval = 1;
      sa.eval_it = kEvalBit | (eval_id & 0x7fffffffu);
      sa.M = per_rank - c0 < ctx->B_local ? per_rank - c0 : ctx->B_local;
      sa.m0 = first + c0;
      sa.inv_B = (float)(1.0 / (double)batch);
      sa.loss_acc = ctx->eval_loss;
      shared_carve(sa, ctx->shbuf, ctx->N_max);
      CK(launch_shared_step(sa, ctx->stream, nullptr, nullptr));
    }
  }
  if (ctx->family == kFamilyRows) {   // the rank's eval paths in chunks of <= B_local rows per step
    const int64_t per_rank = batch / ctx->cfg.world, first = (int64_t)ctx->cfg.rank * per_rank;
    CK(cudaMemsetAsync(ctx->eval_loss, 0, sizeof(double), ctx->stream));
    for (int64_t c0 = 0; c0 < per_rank; c0 += ctx->B_local) {
      RowsArgs ra = rows_args(ctx, per_rank - c0 < ctx->B_local ? per_rank - c0 : ctx->B_local,
                              first + c0);
      ra.eval = 1;
      ra.eval_it = kEvalBit | (eval_id & 0x7fffffffu);
      ra.inv_B = (float)(1.0 / (double)batch);
      ra.loss_acc = ctx->eval_loss;
      CK(launch_rows_forward(ra, ctx->stream, nullptr));
    }
  }
  PassArgs a = pass_args(ctx);
  a.eval = 1;
  a.eval_it = kEvalBit | (eval_id & 0x7fffffffu);
  a.B_local = batch / ctx->cfg.world;
  a.m0 = (int64_t)ctx->cfg.rank * a.B_local;
  a.inv_B = (float)(1.0 / (double)batch);
  a.loss_acc = ctx->eval_loss;
  if (ctx->shared || ctx->family == kFamilyRows) {
  } else if (ctx->family == BSDE_KERNEL_TC) {
    CK(cudaMemsetAsync(ctx->eval_loss, 0, sizeof(double), ctx->stream));
    CK(launch_fwd_tc(a, ctx->stream));   // an evaluation pass stores no path images
  } else {
    CK(cudaMemsetAsync(ctx->eval_loss, 0, sizeof(double), ctx->stream));
    CK(launch_fwd_simt(a, ctx->stream));
  }
  if (!ctx->shared && ctx->cfg.deterministic) {   // the eval batch's own forward grid
    const int tile = ctx->family == BSDE_KERNEL_TC ? 128 : 64;
    const int nt = (int)((a.B_local + tile - 1) / tile);
    CK(launch_det_reduce(a, nt < ctx->sms ? nt : ctx->sms, 0, 1, nt, ctx->stream));
  }
  if (ctx->comm)
    NK(nccl().AllReduce(ctx->eval_loss, ctx->eval_loss, 1, ncclFloat64, ncclSum, ctx->comm,
                        ctx->stream));
  double s;
  CK(cudaMemcpyAsync(&s, ctx->eval_loss, sizeof s, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *loss_out = s / (double)batch;
  return BSDE_OK;
}

int bsde_debug_philox(const bsde_ctx* c, const uint32_t* ctr, const uint32_t key[2],
                      int64_t count, uint32_t* out) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(c);
  if (!ctx || !ctr || !key || !out || count < 1) return fail(ctx, BSDE_EINVAL, "bad argument");
  uint32_t *dc = nullptr, *dout = nullptr;
  CK(cudaMallocAsync((void**)&dc, count * 16, ctx->stream));
  CK(cudaMallocAsync((void**)&dout, count * 16, ctx->stream));
  CK(cudaMemcpyAsync(dc, ctr, count * 16, cudaMemcpyHostToDevice, ctx->stream));
  CK(launch_debug_philox(dc, key[0], key[1], count, dout, ctx->stream));
  CK(cudaMemcpyAsync(out, dout, count * 16, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaFreeAsync(dc, ctx->stream));
  CK(cudaFreeAsync(dout, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}

static int debug_dw_impl(bsde_ctx* ctx, int64_t it, int n, int64_t m0, int64_t count,
                         float* host_out, bool fast) {
  if (!ctx || !host_out || count < 1 || n < 0) return fail(ctx, BSDE_EINVAL, "bad argument");
  float* d_out = nullptr;
  const size_t bytes = (size_t)count * ctx->d * sizeof(float);
  CK(cudaMallocAsync((void**)&d_out, bytes, ctx->stream));
  const float sdt = (float)std::sqrt(ctx->T / ctx->N);
  const uint32_t k0 = (uint32_t)(ctx->cfg.seed & 0xffffffffu), k1 = (uint32_t)(ctx->cfg.seed >> 32);
  if (fast)
    CK(launch_debug_dw_fast((uint32_t)it, n, m0, count, ctx->d, sdt, k0, k1, d_out, ctx->stream));
  else
    CK(launch_debug_dw((uint32_t)it, n, m0, count, ctx->d, sdt, k0, k1, d_out, ctx->stream));
  CK(cudaMemcpyAsync(host_out, d_out, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaFreeAsync(d_out, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}

int bsde_debug_dw(const bsde_ctx* c, int64_t it, int n, int64_t m0, int64_t count,
                  float* host_out) {
  return debug_dw_impl(const_cast<bsde_ctx*>(c), it, n, m0, count, host_out, false);
}

int bsde_debug_dw_fast(const bsde_ctx* c, int64_t it, int n, int64_t m0, int64_t count,
                       float* host_out) {
  return debug_dw_impl(const_cast<bsde_ctx*>(c), it, n, m0, count, host_out, true);
}

int bsde_debug_residuals(const bsde_ctx* c, int64_t m0, int64_t count, float* host_out) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(c);
  if (!ctx || !host_out || m0 < 0 || count < 1 || m0 + count > ctx->B_local)
    return fail(ctx, BSDE_EINVAL, "residual range [%lld, %lld) outside [0, %lld)", (long long)m0,
                (long long)(m0 + count), (long long)(ctx ? ctx->B_local : 0));
  CK(cudaMemcpyAsync(host_out, ctx->Rstore + m0, count * sizeof(float), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return BSDE_OK;
}

int bsde_profile_steps(bsde_ctx* ctx, int steps, float* ms_out, int n_out) {
  if (!ctx || steps < 1 || !ms_out || n_out < 6)
    return fail(ctx, BSDE_EINVAL, "profile_steps: need steps >= 1 and n_out >= 6");
  std::vector<cudaEvent_t> ev(7 * (size_t)steps);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  int rc = BSDE_OK;
  for (int s = 0; s < steps && rc == BSDE_OK; ++s) {
    rc = enqueue_step(ctx, true, &ev[7 * (size_t)s]);
    ctx->host_it += 1;
  }
  if (rc == BSDE_OK) {
    CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 6; ++i) ms_out[i] = 0.0f;
    for (int s = 0; s < steps; ++s)
      for (int i = 0; i < 6; ++i) {
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, ev[7 * (size_t)s + i], ev[7 * (size_t)s + i + 1]));
        ms_out[i] += ms / steps;
      }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

int bsde_debug_phase_clocks(bsde_ctx* ctx, int which, uint64_t* out, int n) {
  if (!ctx || !out || n < 1 || (which != 0 && which != 1) || ctx->family != BSDE_KERNEL_TC ||
      ctx->shared)
    return fail(ctx, BSDE_EINVAL, "debug_phase_clocks: bad argument (tcgen05 path only)");
  unsigned long long* buf = nullptr;
  CK(cudaMalloc(&buf, (size_t)n * sizeof(uint64_t)));
  CK(cudaMemsetAsync(buf, 0, (size_t)n * sizeof(uint64_t), ctx->stream));
  const int64_t np = num_params_at(ctx, ctx->N);
  PassArgs a = pass_args(ctx);
  CK(launch_begin_step(ctx->state, ctx->grad, np, ctx->stream));
  if (which == 0) a.clk = buf;
  CK(launch_fwd_tc(a, ctx->stream));
  if (which == 1) {
    a.clk = buf;
    CK(launch_bwd_tc(a, ctx->stream));
  }
  CK(cudaMemcpyAsync(out, buf, (size_t)n * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(buf);
  return BSDE_OK;
}

int bsde_ipc_export(const bsde_ctx* c, void* out, int64_t bytes) {
  bsde_ctx* ctx = const_cast<bsde_ctx*>(c);
  if (!ctx || !out || bytes < 4 * (int64_t)sizeof(cudaIpcMemHandle_t))
    return fail(ctx, BSDE_EINVAL, "ipc_export: need %d bytes", (int)(4 * sizeof(cudaIpcMemHandle_t)));
  if (ctx->external_ws)
    return fail(ctx, BSDE_EINVAL, "ipc_export: not available with a caller-owned workspace");
  void* bufs[4] = {ctx->grad, ctx->params, ctx->flags, ctx->state};
  cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(out);
  for (int i = 0; i < 4; ++i) CK(cudaIpcGetMemHandle(&h[i], bufs[i]));
  return BSDE_OK;
}

int bsde_fused_opt_enable(bsde_ctx* ctx, const void* handles, int world) {
  if (!ctx) return fail(ctx, BSDE_EINVAL, "ctx is NULL");
  if (world != ctx->cfg.world || world < 1 || world > kMaxPeers)
    return fail(ctx, BSDE_EINVAL, "fused_opt_enable: world=%d (context world %d, at most %d)", world,
                ctx->cfg.world, kMaxPeers);
  if (world > 1 && !handles) return fail(ctx, BSDE_EINVAL, "fused_opt_enable: handles is NULL");
  if (ctx->fused) return fail(ctx, BSDE_ESTATE, "fused optimizer already enabled");
  FusedOptArgs fo{};
  fo.world = world;
  fo.rank = ctx->cfg.rank;
  fo.m = ctx->adam_m;
  fo.v = ctx->adam_v;
  fo.state = ctx->state;
  fo.lr = (float)ctx->cfg.lr;
  fo.beta1 = (float)ctx->cfg.beta1;
  fo.beta2 = (float)ctx->cfg.beta2;
  fo.eps = (float)ctx->cfg.eps;
  const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int q = 0; q < world; ++q) {
    if (q == ctx->cfg.rank) {
      fo.peer_grad[q] = ctx->grad;
      fo.peer_params[q] = ctx->params;
      fo.peer_flags[q] = ctx->flags;
      fo.peer_state[q] = ctx->state;
      continue;
    }
    void* p[4];
    for (int i = 0; i < 4; ++i) {
      CK(cudaIpcOpenMemHandle(&p[i], h[4 * q + i], cudaIpcMemLazyEnablePeerAccess));
      ctx->ipc_open.push_back(p[i]);
    }
    fo.peer_grad[q] = static_cast<float*>(p[0]);
    fo.peer_params[q] = static_cast<float*>(p[1]);
    fo.peer_flags[q] = static_cast<unsigned*>(p[2]);
    fo.peer_state[q] = static_cast<DeviceState*>(p[3]);
  }
  ctx->fo = fo;
  ctx->fused = true;
  if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
  return BSDE_OK;
}

int bsde_launches_per_step(const bsde_ctx* ctx, int* n) {
  if (!ctx || !n) return BSDE_EINVAL;
  *n = ctx->launches;
  return BSDE_OK;
}

const char* bsde_kernel_family(const bsde_ctx* ctx) {
  if (!ctx) return "none";
  if (ctx->shared) return ctx->cfg.precision == BSDE_BF16 ? "shared-tc" : "shared-simt";
  return ctx->family == BSDE_KERNEL_TC ? "tc" : ctx->family == kFamilyRows ? "tc32" : "simt";
}

const char* bsde_last_error(const bsde_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

void bsde_destroy(bsde_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  free_all(ctx);
  delete ctx;
}

}  // extern "C"

extern "C" int bsde_debug_umma(int mode, const float* a, const float* b, float* d_out) {
  bsde_ctx* ctx = nullptr;
  if (mode < 0 || mode > 3 || !a || !b || !d_out) return fail(ctx, BSDE_EINVAL, "debug_umma: bad argument");
  const size_t na = 128 * 112, nb = (mode == 2 ? 128 : 112) * 112, nd = 128 * 112;
  float *da = nullptr, *db = nullptr, *dd = nullptr;
  CK(cudaMalloc(&da, na * 4));
  CK(cudaMalloc(&db, nb * 4));
  CK(cudaMalloc(&dd, nd * 4));
  CK(cudaMemcpy(da, a, na * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b, nb * 4, cudaMemcpyHostToDevice));
  CK(launch_umma_test(mode, da, db, dd, 0));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(d_out, dd, nd * 4, cudaMemcpyDeviceToHost));
  cudaFree(da);
  cudaFree(db);
  cudaFree(dd);
  return BSDE_OK;
}
