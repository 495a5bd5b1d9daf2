"""Python face of libbsde.so: one object per GPU/rank wrapping a bsde_ctx.

Marshalling only — every step of the training iteration runs in the CUDA
kernels behind include/bsde.h.  PyTorch is used for the device's current
stream and for torch.distributed (broadcast of the NCCL unique id).
"""
import ctypes

import numpy as np

from . import _lib
from ._lib import BSDEError

FORMULATIONS = {"per_step": 0, "shared": 1}
ARCHS = {"fc": 0, "resnet": 1, "nais": 2}
PROBLEMS = {"heat": _lib.HEAT, "hjb": _lib.HJB, "allen_cahn": _lib.ALLEN_CAHN,
            "black_scholes": _lib.BLACK_SCHOLES}
PRECISIONS = {"fp32": _lib.FP32, "bf16": _lib.BF16}
KERNELS = {"auto": _lib.KERNEL_AUTO, "simt": _lib.KERNEL_SIMT, "tc": _lib.KERNEL_TC}
PROLONG = {"copy": _lib.PROLONG_COPY, "interp": _lib.PROLONG_INTERP}


def _fptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    rc = _lib.lib().bsde_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if rc:
        raise BSDEError(rc, _lib.lib().bsde_last_error(None).decode())
    return buf.raw


def debug_umma(mode, a, b):
    """One bf16 tcgen05 MMA (M=128, N=112) in the given operand-major mode."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    out = np.empty((128, 112), np.float32)
    rc = _lib.lib().bsde_debug_umma(int(mode), _fptr(a), _fptr(b), _fptr(out))
    if rc:
        raise BSDEError(rc, _lib.lib().bsde_last_error(None).decode())
    return out


def step_size(d, w):
    return 2 * d * w + w * w + 2 * w + d


def workspace_bytes(problem, d, N, width, batch, *, precision="fp32", kernel="auto", world=1,
                    max_levels=0, formulation="per_step", arch="fc", layers=4, sharded_adam=False):
    """bsde_workspace_bytes: device bytes of a context (no GPU needed)."""
    L = _lib.lib()
    cfg = _lib.Config()
    L.bsde_config_default(ctypes.byref(cfg))
    cfg.batch_global, cfg.world = int(batch), int(world)
    cfg.precision = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
    cfg.kernel = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    cfg.max_levels = int(max_levels)
    cfg.formulation, cfg.arch = FORMULATIONS[formulation], ARCHS[arch]
    cfg.sharded_adam = int(bool(sharded_adam))
    nw = int(layers) if formulation == "shared" else 2
    widths = (ctypes.c_int * nw)(*([int(width)] * nw))
    out = ctypes.c_size_t()
    p = PROBLEMS[problem] if isinstance(problem, str) else int(problem)
    rc = L.bsde_workspace_bytes(p, int(d), int(N), widths, nw, ctypes.byref(cfg), ctypes.byref(out))
    if rc:
        raise BSDEError(rc, L.bsde_last_error(None).decode())
    return out.value


class BSDE:
    """bsde_create(problem, d, N, T, widths) + the step / level / introspection calls."""

    def __init__(self, problem, d, N, T, width, batch, *, lr=1e-2, seed=0, precision="fp32",
                 kernel="auto", x0=0.0, lam=1.0, prolong="copy", max_levels=0, device=0,
                 stream=None, rank=0, world=1, nccl_id=None, use_graph=True, beta1=0.9,
                 beta2=0.999, eps=1e-8, zero_head=None, coupled_paths=False,
                 formulation="per_step", arch="fc", layers=4, sharded_adam=False,
                 workspace=None, deterministic=False, zN=False, keep_adam=False):
        """stream: a torch.cuda.Stream, a raw cudaStream_t (int), or None (a new
        torch stream on `device`, kept in self.stream).  zero_head: R7b, defaults
        to True for Allen-Cahn.  coupled_paths: every level draws the finest grid's
        (N·2^max_levels) Brownian path, summed per coarse step (NEXT-3).
        keep_adam: at a level change prolong the Adam moments like the parameters and
        keep t (R14b) instead of resetting them (R14).
        formulation="shared": the paper's own method (one tanh network u(t, x) of
        `layers` layers of `width`, arch "fc" | "resnet", Eq. 6 loss; NEXT-1)."""
        L = _lib.lib()
        cfg = _lib.Config()
        L.bsde_config_default(ctypes.byref(cfg))
        cfg.batch_global = int(batch)
        cfg.x0, cfg.lam = float(x0), float(lam)
        cfg.lr, cfg.beta1, cfg.beta2, cfg.eps = float(lr), float(beta1), float(beta2), float(eps)
        cfg.seed = int(seed)
        self.seed = int(seed)
        cfg.precision = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
        cfg.kernel = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
        cfg.prolong_mode = PROLONG[prolong] if isinstance(prolong, str) else int(prolong)
        if keep_adam:
            cfg.prolong_mode |= _lib.PROLONG_KEEP_ADAM
        cfg.max_levels = int(max_levels)
        cfg.device = int(device)
        self.stream = None
        if stream is None:
            import torch
            if torch.cuda.is_available():
                self.stream = torch.cuda.Stream(device=device)
                stream = self.stream.cuda_stream
        elif not isinstance(stream, int):
            self.stream = stream
            stream = stream.cuda_stream
        cfg.stream = stream or None
        if zero_head is None:
            zero_head = (problem == "allen_cahn" or problem == _lib.ALLEN_CAHN)
        cfg.init_zero_head = int(bool(zero_head))
        self.zero_head = bool(zero_head)
        cfg.rank, cfg.world = int(rank), int(world)
        self._nccl_id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        cfg.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p) if nccl_id else None
        cfg.use_graph = int(bool(use_graph))
        cfg.coupled_paths = int(bool(coupled_paths))
        cfg.formulation = FORMULATIONS[formulation]
        cfg.sharded_adam = int(bool(sharded_adam))
        self._sharded, self._fused = bool(sharded_adam), False
        cfg.deterministic = int(bool(deterministic))
        cfg.shared_zN = int(bool(zN))
        if workspace is not None:   # caller-owned device memory (a torch tensor), kept alive
            self._workspace = workspace
            cfg.workspace = workspace.data_ptr()
            cfg.workspace_bytes = workspace.numel() * workspace.element_size()
        cfg.arch = ARCHS[arch]
        self.formulation, self.arch, self.layers = formulation, arch, int(layers)
        self.problem = PROBLEMS[problem] if isinstance(problem, str) else int(problem)
        self.d, self.w, self.T, self.batch = int(d), int(width), float(T), int(batch)
        self.rank, self.world = int(rank), int(world)
        nw = self.layers if formulation == "shared" else 2
        widths = (ctypes.c_int * nw)(*([int(width)] * nw))
        h = ctypes.c_void_p()
        rc = L.bsde_create(self.problem, self.d, int(N), self.T, widths, nw, ctypes.byref(cfg),
                           ctypes.byref(h))
        if rc:
            raise BSDEError(rc, L.bsde_last_error(None).decode())
        self._h = h
        self._L = L

    @classmethod
    def distributed(cls, problem, d, N, T, width, batch, **kw):
        """One context per rank of the default torch.distributed group; rank 0
        creates the NCCL unique id and broadcasts it."""
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        return cls(problem, d, N, T, width, batch, rank=rank, world=world, nccl_id=obj[0], **kw)

    # ------------------------------------------------------------------ core
    def _ck(self, rc):
        if rc:
            raise BSDEError(rc, self._L.bsde_last_error(self._h).decode())

    def train_step(self, sync=True):
        """One iteration (a1-a8).  sync=True returns the pre-update loss."""
        if not sync:
            self._ck(self._L.bsde_train_step(self._h, None))
            return None
        loss = ctypes.c_double()
        self._ck(self._L.bsde_train_step(self._h, ctypes.byref(loss)))
        return loss.value

    def compute_grad(self):
        loss = ctypes.c_double()
        self._ck(self._L.bsde_compute_grad(self._h, ctypes.byref(loss)))
        return loss.value

    def prolongate(self, level):
        self._ck(self._L.bsde_prolongate(self._h, int(level)))

    def y0(self):
        v = ctypes.c_double()
        self._ck(self._L.bsde_y0(self._h, ctypes.byref(v)))
        return v.value

    def eval_loss(self, eval_id=0, batch=None):
        v = ctypes.c_double()
        self._ck(self._L.bsde_eval_loss(self._h, int(eval_id), int(batch or self.batch),
                                        ctypes.byref(v)))
        return v.value

    # ------------------------------------------------------------------ state
    @property
    def N(self):
        n = ctypes.c_int()
        self._ck(self._L.bsde_current_steps(self._h, ctypes.byref(n)))
        return n.value

    def num_params(self):
        n = ctypes.c_int64()
        self._ck(self._L.bsde_num_params(self._h, ctypes.byref(n)))
        return n.value

    def get_params(self):
        a = np.empty(self.num_params(), np.float32)
        self._ck(self._L.bsde_get_params(self._h, _fptr(a), a.size))
        return a

    def set_params(self, p):
        a = np.ascontiguousarray(p, dtype=np.float32)
        self._ck(self._L.bsde_set_params(self._h, _fptr(a), a.size))

    def get_grads(self):
        a = np.empty(self.num_params(), np.float32)
        self._ck(self._L.bsde_get_grads(self._h, _fptr(a), a.size))
        return a

    def get_adam_state(self):
        n = self.num_params()
        m, v, t = np.empty(n, np.float32), np.empty(n, np.float32), ctypes.c_int64()
        self._ck(self._L.bsde_get_adam_state(self._h, _fptr(m), _fptr(v), n, ctypes.byref(t)))
        return m, v, t.value

    def set_adam_state(self, m, v, t):
        m = np.ascontiguousarray(m, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        self._ck(self._L.bsde_set_adam_state(self._h, _fptr(m), _fptr(v), m.size, int(t)))

    # ------------------------------------------------------------------ checkpoint
    def save_checkpoint(self, path):
        """Flat named arrays: parameters, Adam m, v, t and the
        Philox iteration (the paths of every later iteration follow from it, R8/R9).
        np.savez; bit-exact round trip through load_checkpoint.  A rank of a sharded
        optimizer (sharded_adam or the fused NEXT-4 kernel, world > 1) holds the Adam
        moments of its own shard only, so its checkpoint would not restore the others:
        refused."""
        if self.world > 1 and (self._sharded or self._fused):
            raise BSDEError(-5, "save_checkpoint: Adam state is sharded over the ranks "
                                "(sharded_adam / fused optimizer), a single rank cannot save it")
        m, v, t = self.get_adam_state()
        np.savez(path, params=self.get_params(), adam_m=m, adam_v=v, adam_t=np.int64(t),
                 iteration=np.int64(self.iteration), N=np.int64(self.N),
                 seed=np.uint64(self.seed),
                 manifest=np.array(["params", "adam_m", "adam_v", "adam_t", "iteration", "N",
                                    "seed"]))

    def load_checkpoint(self, path):
        """Restore a checkpoint written by save_checkpoint into a context of the same
        shape (problem, d, widths and the current N)."""
        z = np.load(path)
        if int(z["seed"]) != self.seed:   # the paths of later iterations depend on it (R8)
            raise ValueError("checkpoint seed %d != context seed %d" % (int(z["seed"]), self.seed))
        if int(z["N"]) != self.N or z["params"].size != self.num_params():
            raise ValueError("checkpoint has N=%d and %d parameters; this context N=%d, %d"
                             % (int(z["N"]), z["params"].size, self.N, self.num_params()))
        self.set_params(z["params"])
        self.set_adam_state(z["adam_m"], z["adam_v"], int(z["adam_t"]))
        self.iteration = int(z["iteration"])

    @property
    def iteration(self):
        v = ctypes.c_int64()
        self._ck(self._L.bsde_get_iteration(self._h, ctypes.byref(v)))
        return v.value

    @iteration.setter
    def iteration(self, it):
        self._ck(self._L.bsde_set_iteration(self._h, int(it)))

    def enable_fused_optimizer(self):
        """NEXT-4: switch the optimizer to the single peer-memory kernel (reduce-scatter,
        sharded Adam, all-gather; fused_opt.cu).  Collective: with world > 1 every rank
        calls it after torch.distributed is initialised (the 256-byte CUDA IPC handles
        are exchanged with all_gather_object); at world = 1 the peer is the context."""
        world = self.world
        if world > 1:
            import torch.distributed as dist
            buf = ctypes.create_string_buffer(256)
            self._ck(self._L.bsde_ipc_export(self._h, ctypes.cast(buf, ctypes.c_void_p), 256))
            parts = [None] * world
            dist.all_gather_object(parts, buf.raw)
            allh = ctypes.create_string_buffer(b"".join(parts), 256 * world)
            self._ck(self._L.bsde_fused_opt_enable(self._h, ctypes.cast(allh, ctypes.c_void_p), world))
        else:
            self._ck(self._L.bsde_fused_opt_enable(self._h, None, 1))
        self._fused = True

    def launches_per_step(self):
        n = ctypes.c_int()
        self._ck(self._L.bsde_launches_per_step(self._h, ctypes.byref(n)))
        return n.value

    @property
    def family(self):
        return self._L.bsde_kernel_family(self._h).decode()

    # ------------------------------------------------------------------ test hooks
    def debug_philox(self, ctr, key):
        ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
        key = np.ascontiguousarray(key, np.uint32).reshape(2)
        out = np.empty_like(ctr)
        P = ctypes.POINTER(ctypes.c_uint32)
        self._ck(self._L.bsde_debug_philox(self._h, ctr.ctypes.data_as(P), key.ctypes.data_as(P),
                                           ctr.shape[0], out.ctypes.data_as(P)))
        return out

    def debug_dw(self, it, n, m0, count, fast=False):
        out = np.empty((count, self.d), np.float32)
        fn = self._L.bsde_debug_dw_fast if fast else self._L.bsde_debug_dw
        self._ck(fn(self._h, int(it), int(n), int(m0), int(count), _fptr(out)))
        return out

    PHASES = ("begin", "fwd", "bwd", "allreduce", "check", "adam")

    def profile_steps(self, steps):
        """Mean per-phase milliseconds over `steps` eager iterations (CUDA events)."""
        out = np.zeros(6, np.float32)
        self._ck(self._L.bsde_profile_steps(self._h, int(steps), _fptr(out), 6))
        return dict(zip(self.PHASES, out.tolist()))

    def debug_phase_clocks(self, which, n=1024):
        """clock64() stamps of CTA 0 (16 per step / item; 0 = unused), see tc.cu CLK."""
        out = np.zeros(n, np.uint64)
        self._ck(self._L.bsde_debug_phase_clocks(
            self._h, int(which), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n))
        return out.reshape(-1, 16)

    def debug_residuals(self, m0, count):
        out = np.empty(count, np.float32)
        self._ck(self._L.bsde_debug_residuals(self._h, int(m0), int(count), _fptr(out)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._L.bsde_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
