"""Sample-sharded CGLS across ranks (the C4 row).

T stacks the rank-local row blocks T_g (each rank owns a contiguous slice of
the samples and a device-resident operator built from it); coefficient-space
vectors x, p, s are replicated.  One CGNR iteration (solver.cpp:70-88) then
needs exactly two exchanges:

    q_g = T_g p                       local
    qq  = sum_g ||q_g||^2             allreduce of 1 number
    r_g -= alpha q_g ; x += alpha p   local
    s   = sum_g T_g^* r_g             allreduce of N_c complex (NCCL over NVLink)
    gamma', beta, p = s + beta p      local, replicated

Summing coefficient-space adjoint partials equals summing the oversampled
grids by linearity and is (sigma^dim =) 4x smaller.

Two implementations of the same iteration:
  * the product path -- `Communicator` + `ShardedSession` /
    `solve_least_squares_sharded`: the library runs the loop resident on the
    GPU and issues both sums as NCCL allreduces on its own stream
    (gs_cgls_begin_sharded / gs_solve_least_squares_sharded, include/gs_b200.h);
    no host round trip per iteration;
  * `cgls_sharded` / `ShardedCGLS`: the loop written against three callables,
    so the CPU tests drive the oracle with gloo through the same algebra.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


@dataclass
class ShardedStats:
    iterations: int = 0
    residual: float = 0.0
    history: list = field(default_factory=list)
    converged: bool = False


def cgls_sharded(apply_forward, apply_adjoint, b_local, x0, allreduce_sum, norm2, max_iterations, tolerance):
    """CGNR of solver.cpp:19-91 over sharded rows.

    apply_forward(x) -> local rows; apply_adjoint(r_local) -> this rank's partial
    T_g^* r_g; allreduce_sum(v) sums a vector (or 1-element vector) over ranks in
    place and returns it; norm2(v) -> float; b_local already carries sqrt(mu).
    x0 is the replicated initial guess (or a zero vector)."""
    if not (tolerance > 0):
        raise ValueError("tolerance must be positive")
    st = ShardedStats()
    s = allreduce_sum(apply_adjoint(b_local))
    ref = math.sqrt(norm2(s))
    x = x0.clone() if hasattr(x0, "clone") else x0.copy()
    if ref == 0.0:  # solver.cpp:43-48
        st.converged = True
        st.history = [0.0]
        return x * 0, st
    r = b_local - apply_forward(x)
    s = allreduce_sum(apply_adjoint(r))
    gamma = norm2(s)
    st.history.append(math.sqrt(gamma) / ref)
    if st.history[-1] <= tolerance:
        st.converged = True
        st.residual = st.history[-1]
        return x, st
    p = s
    for it in range(1, max_iterations + 1):
        q = apply_forward(p)
        qq = _scalar_allreduce(norm2(q), allreduce_sum, q)
        if qq == 0.0:
            break
        alpha = gamma / qq
        x = x + alpha * p
        r = r - alpha * q
        s = allreduce_sum(apply_adjoint(r))
        gnew = norm2(s)
        st.iterations = it
        st.history.append(math.sqrt(gnew) / ref)
        if st.history[-1] <= tolerance:
            st.converged = True
            break
        beta = gnew / gamma
        gamma = gnew
        p = s + beta * p
    st.residual = st.history[-1]
    return x, st


class ShardedCGLS:
    """The same iteration split into begin() (preamble, solver.cpp:28-68) and
    step(k) (k loop bodies), for timing fixed iteration counts."""

    def __init__(self, apply_forward, apply_adjoint, b_local, x0, allreduce_sum, norm2):
        self.f, self.a, self.ar, self.n2 = apply_forward, apply_adjoint, allreduce_sum, norm2
        s = self.ar(self.a(b_local))
        self.ref = math.sqrt(self.n2(s))
        self.x = x0.clone()
        self.r = b_local - self.f(self.x)
        self.s = self.ar(self.a(self.r))
        self.gamma = self.n2(self.s)
        self.p = self.s
        self.history = [math.sqrt(self.gamma) / self.ref if self.ref else 0.0]
        self.active = self.ref != 0.0

    def step(self, k):
        for _ in range(k):
            if not self.active:
                return
            q = self.f(self.p)
            qq = _scalar_allreduce(self.n2(q), self.ar, q)
            if qq == 0.0:
                self.active = False
                return
            alpha = self.gamma / qq
            self.x = self.x + alpha * self.p
            self.r = self.r - alpha * q
            self.s = self.ar(self.a(self.r))
            gnew = self.n2(self.s)
            self.history.append(math.sqrt(gnew) / self.ref)
            beta = gnew / self.gamma
            self.gamma = gnew
            self.p = self.s + beta * self.p


def _scalar_allreduce(v, allreduce_sum, like):
    if hasattr(like, "new_tensor"):
        t = like.new_tensor([v], dtype=like.real.dtype if like.is_complex() else like.dtype)
        return float(allreduce_sum(t).item())
    import numpy as np
    return float(allreduce_sum(np.array([v]))[0])


def shard_range(total, rank, world):
    """Contiguous [lo, hi) of `total` samples owned by `rank`."""
    return rank * total // world, (rank + 1) * total // world


def torch_collectives(group=None):
    """allreduce_sum / norm2 over torch.distributed (NCCL for CUDA tensors)."""
    import torch
    import torch.distributed as dist

    def allreduce_sum(v):
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
        return v

    def norm2(v):
        return float(torch.sum(v.real * v.real + v.imag * v.imag).item()) if v.is_complex() else \
            float(torch.sum(v * v).item())

    return allreduce_sum, norm2


# ------------------------------------------------------------------ library (NCCL) path
class Communicator:
    """NCCL communicator owned by libgs_b200.so (gs_comm_init).  Rank 0 makes
    the unique id; `from_torch` ships it with torch.distributed (any backend)."""

    def __init__(self, nranks, rank, uid: bytes, device=0):
        import ctypes as C

        from . import _check, load_library
        L = load_library()
        L.gs_comm_init.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.gs_comm_destroy.argtypes = [C.c_void_p]
        h = C.c_void_p()
        _check(L.gs_comm_init(int(nranks), int(rank), uid, int(device), C.byref(h)))
        self._h, self.nranks, self.rank, self.device = h, nranks, rank, device

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        from . import _check, load_library
        buf = (C.c_ubyte * 128)()
        _check(load_library().gs_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_torch(cls, device=0, group=None):
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        obj = [cls.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(world, rank, obj[0], device)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            from . import load_library
            load_library().gs_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedSession:
    """gs_cgls_begin_sharded / step / finish: the resident CGLS loop of
    solver.cpp:19-91 over this rank's rows, both sums by NCCL on the device."""

    def __init__(self, op, comm: Communicator, samples_local, tolerance=1e-300, history_capacity=2,
                 initial_guess=None, stream=None):
        import ctypes as C

        from . import _check, _ptr_len, _stream_ptr, load_library
        L = load_library()
        L.gs_cgls_begin_sharded.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_double,
                                            C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
        self.op = op
        p, n, self._keep = _ptr_len(samples_local)
        x0p = None
        if initial_guess is not None:
            x0p, _, self._keep0 = _ptr_len(initial_guess)
        self._cap = max(2, history_capacity)
        h = C.c_void_p()
        _check(L.gs_cgls_begin_sharded(op.handle, comm.handle, p, n, x0p, float(tolerance), self._cap,
                                       _stream_ptr(stream), C.byref(h)))
        self._h = h

    def step(self, iterations, stream=None):
        from . import _check, _stream_ptr, load_library
        _check(load_library().gs_cgls_step(self._h, int(iterations), _stream_ptr(stream)))

    def result(self, stream=None):
        import numpy as np

        from . import CglsSession
        return CglsSession.result(self, None, stream)

    def close(self):
        if getattr(self, "_h", None):
            from . import load_library
            load_library().gs_cgls_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_least_squares_sharded(op, comm: Communicator, samples_local, max_iterations=0, tolerance=1e-10,
                                initial_guess=None, stream=None):
    """gs::solve_least_squares over the rows of all ranks (every rank passes its
    own operator / raw samples; x and the stats come back replicated)."""
    import ctypes as C

    import numpy as np

    from . import SolveStats, _check, _ptr_len, _Stats, _stream_ptr, load_library
    L = load_library()
    L.gs_solve_least_squares_sharded.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int,
                                                 C.c_double, C.c_void_p, C.POINTER(_Stats),
                                                 C.POINTER(C.c_double), C.c_void_p]
    p, n, keep = _ptr_len(samples_local)
    x0p = None
    keep0 = None
    if initial_guess is not None:
        x0p, _, keep0 = _ptr_len(initial_guess)
    B = op.batch
    mi = max_iterations if max_iterations > 0 else 2 * op.cols()
    x = np.empty(op.cols() * B, np.complex128)
    stats = (_Stats * B)()
    hist = np.zeros(B * (mi + 1), np.float64)
    _check(L.gs_solve_least_squares_sharded(op.handle, comm.handle, p, n, x0p, int(max_iterations), float(tolerance),
                                            x.ctypes.data, stats, hist.ctypes.data_as(C.POINTER(C.c_double)),
                                            _stream_ptr(stream)))
    out = [SolveStats(s.iterations, s.residual, hist[b * (mi + 1):b * (mi + 1) + s.iterations + 1].tolist(),
                      bool(s.converged)) for b, s in enumerate(stats)]
    return (x, out[0]) if B == 1 else (x, out)
