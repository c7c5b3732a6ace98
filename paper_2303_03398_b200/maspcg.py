"""Thin Python binding of libmaspcg (include/maspcg.h) -- argument marshalling only.

Every step of the solve runs in the CUDA kernels of libmaspcg.so; this module
only converts torch tensors / numpy arrays to pointers, passes the caller's
CUDA stream, allocates the workspace as a torch uint8 tensor and broadcasts
the NCCL unique id through a torch.distributed process group.  There is no
CPU fallback: if libmaspcg.so is missing or no GPU is visible, calls raise.

Names mirror the C ABI: ``maspcg_create`` -> ``Solver.__init__``,
``maspcg_set_coefficients`` -> ``Solver.set_coefficients``, ``maspcg_set_bc_r``
-> ``Solver.set_bc_r``, ``maspcg_solve`` -> ``Solver.solve``, ``maspcg_apply`` ->
``Solver.apply``, and so on; the raw functions are reachable as ``lib().maspcg_*``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libmaspcg.so")

OK, NOT_CONVERGED = 0, 1
E_INVALID, E_STATE, E_SINGULAR, E_BREAKDOWN, E_CUDA, E_NCCL, E_NOMEM = -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "OK", 1: "NOT_CONVERGED", -1: "E_INVALID", -2: "E_STATE", -3: "E_SINGULAR",
                -4: "E_BREAKDOWN", -5: "E_CUDA", -6: "E_NCCL", -7: "E_NOMEM"}
BC_DIRICHLET, BC_NEUMANN0 = 0, 1
WALL_NO_SLIP, WALL_FREE_SLIP = 0, 1
MEAN_ARITHMETIC, MEAN_HARMONIC = 0, 1
OPT_CHUNK, OPT_USE_GRAPHS, OPT_TIMING, OPT_PATH, OPT_ARITH, OPT_TMA, OPT_VEC, OPT_PDL = 1, 2, 3, 4, 5, 6, 7, 8
OPT_FUSE_HALO = 9
OPT_L2_KEEP = 10
OPT_DEVICE_LOOP = 11
ARITH_EXACT, ARITH_FAST = 0, 1
PATH_AUTO, PATH_THREE_KERNELS, PATH_FUSED = 0, 1, 2


class MaspcgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Info(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("bnorm", ctypes.c_double), ("rnorm", ctypes.c_double),
                ("rel_resid", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_longlong), ("solves", ctypes.c_longlong),
                ("iterations", ctypes.c_longlong), ("matvec_ms", ctypes.c_double),
                ("matvec_launches", ctypes.c_longlong), ("update_ms", ctypes.c_double),
                ("update_launches", ctypes.c_longlong), ("pupdate_ms", ctypes.c_double),
                ("pupdate_launches", ctypes.c_longlong), ("comm_ms", ctypes.c_double), ("halo_ms", ctypes.c_double),
                ("comm_launches", ctypes.c_longlong), ("path", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# exported symbol -> (argtypes, restype); the list is also the ABI the tests check against include/maspcg.h
_V, _I, _D, _SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
SIGNATURES = {
    "maspcg_get_unique_id": ([_V], _I),
    "maspcg_create": ([_I, _I, _I, _I, _I, _V, _I, ctypes.POINTER(_V)], _I),
    "maspcg_destroy": ([_V], _I),
    "maspcg_last_error": ([_V], ctypes.c_char_p),
    "maspcg_set_grid": ([_V, _V, _V, _V], _I),
    "maspcg_local_extent": ([_V, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "maspcg_workspace_bytes": ([_V], _SZ),
    "maspcg_set_workspace": ([_V, _V, _SZ], _I),
    "maspcg_set_coefficients": ([_V, _V, _V, _V, _V, _V], _I),
    "maspcg_set_coefficients_host": ([_V, _V, _V, _V, _V, _V], _I),
    "maspcg_set_coefficients_from_fields": ([_V, _V, _D, _I, _I, _V, _D, _V], _I),
    "maspcg_set_bc_r": ([_V, _I, _V, _I, _V, _V], _I),
    "maspcg_set_bc_r_host": ([_V, _I, _V, _I, _V, _V], _I),
    "maspcg_solve": ([_V, _V, _V, _D, _I, _V, ctypes.POINTER(Info), _V], _I),
    "maspcg_solve_host": ([_V, _V, _V, _D, _I, _V, ctypes.POINTER(Info), _V], _I),
    "maspcg_apply": ([_V, _V, _V, _V], _I),
    "maspcg_sts_step": ([_V, _V, _D, _I, _V], _I),
    "maspcg_sts_dt_limit": ([_V, ctypes.POINTER(_D), _V], _I),
    "maspcg_get_operator": ([_V, _V, _V, _V, _V, _V], _I),
    "maspcg_set_option": ([_V, _I, ctypes.c_longlong], _I),
    "maspcg_get_stats": ([_V, ctypes.POINTER(Stats)], _I),
    "maspcg_reset_stats": ([_V], _I),
    "maspcg_version": ([], ctypes.c_char_p),
    "maspcg_loopback_group_create": ([_I, ctypes.POINTER(_V)], _I),
    "maspcg_loopback_group_destroy": ([_V], _I),
    "maspcg_create_loopback": ([_I, _I, _I, _I, _I, _V, _I, ctypes.POINTER(_V)], _I),
    "maspcg_vv_workspace_bytes": ([_V], _SZ),
    "maspcg_vv_set_workspace": ([_V, _V, _SZ], _I),
    "maspcg_vv_set_coefficients": ([_V, _V, _V, _V], _I),
    "maspcg_vv_set_bc_r": ([_V, _I, _V, _I, _V, _V], _I),
    "maspcg_vv_apply": ([_V, _V, _V, _V], _I),
    "maspcg_vv_solve": ([_V, _V, _V, _D, _I, _V, ctypes.POINTER(Info), _V], _I),
    "maspcg_vv_get_diag": ([_V, _V, _V], _I),
    "maspcg_aniso_workspace_bytes": ([_V], _SZ),
    "maspcg_aniso_set_workspace": ([_V, _V, _SZ], _I),
    "maspcg_set_aniso_coefficients": ([_V, _V, _V, _V, _V], _I),
    "maspcg_aniso_get_operator": ([_V, _V, _V, _V, _V, _V], _I),
    "maspcg_create_peer": ([_I, _I, _I, _I, _I, _V, _I, ctypes.POINTER(_V)], _I),
    "maspcg_peer_export": ([_V, _I, _V], _I),
    "maspcg_peer_import": ([_V, _I, _I, _V], _I),
}
P2P_HANDLE_BYTES = 80

_lib = None


def lib() -> ctypes.CDLL:
    """Load libmaspcg.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2303_03398_b200.build` "
                              "(nvcc, sm_100a); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _ptr(t) -> int | None:
    """Device or host pointer of a torch tensor / numpy array (must be contiguous float64)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        if t.dtype != np.float64 or not t.flags.c_contiguous:
            raise TypeError("numpy arrays must be C-contiguous float64")
        return t.ctypes.data
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"expected a torch.Tensor or numpy array, got {type(t)}")
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("tensors must be contiguous float64")
    return t.data_ptr()


def _stream(stream=None) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class Solver:
    """One rank's handle on the distributed solve (maspcg_create ... maspcg_destroy).

    ``group``: a torch.distributed process group (or None for the default group when
    torch.distributed is initialised with world size > 1); its size is the number of
    GPUs the phi-slabs are spread over.  ``device``: the CUDA device index (default:
    torch's current device)."""

    def __init__(self, nr: int, nt: int, np_: int, rf, tf, pf, *, group=None, device: int | None = None,
                 chunk: int = 16, loopback: "tuple[LoopbackGroup, int] | None" = None,
                 force_comm: bool = False, comm: str = "nccl"):
        """comm: "nccl" (NCCL send/recv and all-gathers) or "peer" (maspcg_create_peer: exchanges as
        kernels storing into the peers' workspaces over NVLink; with `loopback` the ranks share this
        process, otherwise the workspaces are mapped by CUDA IPC handles exchanged over `group`)."""
        import torch
        import torch.distributed as dist
        self._L = lib()
        self.ctx = None
        self.comm = comm
        self.group = group
        if not torch.cuda.is_available():
            raise MaspcgError(E_CUDA, "no CUDA device visible (libmaspcg has no CPU fallback)")
        if loopback is not None:
            lgroup, self.rank = loopback
            self.nranks = lgroup.nranks
        elif dist.is_available() and dist.is_initialized() and (group is not None or dist.get_world_size() > 1):
            self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.nranks = 0, 1
        self.device = torch.cuda.current_device() if device is None else int(device)
        uid = None
        self._ipc = comm == "peer" and loopback is None and self.nranks > 1
        if comm == "peer":
            ctx = ctypes.c_void_p()
            st = self._L.maspcg_create_peer(nr, nt, np_, self.rank, self.nranks,
                                            loopback[0].handle if loopback is not None else None, self.device,
                                            ctypes.byref(ctx))
            if st != OK:
                raise MaspcgError(st, self._L.maspcg_last_error(None).decode())
            self._init_after_create(ctx, nr, nt, np_, rf, tf, pf, chunk)
            return
        if loopback is not None:
            ctx = ctypes.c_void_p()
            st = self._L.maspcg_create_loopback(nr, nt, np_, self.rank, self.nranks, lgroup.handle, self.device,
                                                ctypes.byref(ctx))
            if st != OK:
                raise MaspcgError(st, self._L.maspcg_last_error(None).decode())
            self._init_after_create(ctx, nr, nt, np_, rf, tf, pf, chunk)
            return
        if self.nranks == 1 and force_comm:
            # one rank with a real NCCL communicator: the multi-rank code path (halo send/recv to itself,
            # all-gathers of one) on one GPU -- the periodic wrap then goes through NCCL
            uid = ctypes.create_string_buffer(128)
            self._check(self._L.maspcg_get_unique_id(uid), None)
        elif self.nranks > 1:
            buf = ctypes.create_string_buffer(128)
            if self.rank == 0:
                self._check(self._L.maspcg_get_unique_id(buf), None)
            obj = [buf.raw if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        ctx = ctypes.c_void_p()
        st = self._L.maspcg_create(nr, nt, np_, self.rank, self.nranks, uid, self.device, ctypes.byref(ctx))
        if st != OK:
            raise MaspcgError(st, self._L.maspcg_last_error(None).decode())
        self._init_after_create(ctx, nr, nt, np_, rf, tf, pf, chunk)

    def _init_after_create(self, ctx, nr, nt, np_, rf, tf, pf, chunk):
        import torch
        self.ctx = ctx
        self.nr, self.nt, self.np = nr, nt, np_
        k0, nloc = ctypes.c_int(), ctypes.c_int()
        self._L.maspcg_local_extent(ctx, ctypes.byref(k0), ctypes.byref(nloc))
        self.k0, self.nloc = k0.value, nloc.value
        self.set_grid(rf, tf, pf)
        nbytes = self._L.maspcg_workspace_bytes(ctx)
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        base = self.workspace.data_ptr()
        off = (-base) % 256
        self._check(self._L.maspcg_set_workspace(ctx, base + off, nbytes))
        if getattr(self, "_ipc", False):
            self._peer_exchange(0)
        self.set_option(OPT_CHUNK, chunk)

    def _peer_exchange(self, region: int):
        """Peer mode across processes: all-gather the CUDA IPC handles of workspace `region` over the
        process group and map every peer's (maspcg_peer_export / maspcg_peer_import)."""
        import torch.distributed as dist
        buf = ctypes.create_string_buffer(P2P_HANDLE_BYTES)
        self._check(self._L.maspcg_peer_export(self.ctx, region, buf))
        allh = [None] * self.nranks
        dist.all_gather_object(allh, buf.raw, group=self.group)
        for r, h in enumerate(allh):
            if r != self.rank:
                hb = ctypes.create_string_buffer(h, P2P_HANDLE_BYTES)
                self._check(self._L.maspcg_peer_import(self.ctx, region, r, hb))
        dist.barrier(group=self.group)

    # ---------------------------------------------------------------- plumbing
    def _check(self, st: int, ctx="self", ok=(OK,)):
        if st not in ok:
            msg = self._L.maspcg_last_error(self.ctx if ctx == "self" else ctx)
            raise MaspcgError(st, (msg or b"").decode())
        return st

    def close(self):
        if getattr(self, "ctx", None):
            self._L.maspcg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def local_shape(self):
        return (self.nloc, self.nt, self.nr)

    # ---------------------------------------------------------------- C-ABI mirrors
    def set_grid(self, rf, tf, pf):
        rf, tf, pf = (np.ascontiguousarray(a, dtype=np.float64) for a in (rf, tf, pf))
        assert rf.size == self.nr + 1 and tf.size == self.nt + 1 and pf.size == self.np + 1
        self._check(self._L.maspcg_set_grid(self.ctx, _ptr(rf), _ptr(tf), _ptr(pf)))

    def set_option(self, opt: int, value: int):
        self._check(self._L.maspcg_set_option(self.ctx, opt, int(value)))

    def set_coefficients(self, kr, kt, kp, s, stream=None):
        """Device tensors (maspcg_set_coefficients) or numpy arrays (maspcg_set_coefficients_host)."""
        host = isinstance(kr, np.ndarray)
        fn = self._L.maspcg_set_coefficients_host if host else self._L.maspcg_set_coefficients
        self._check(fn(self.ctx, _ptr(kr), _ptr(kt), _ptr(kp), _ptr(s), _stream(stream)))

    def set_coefficients_from_fields(self, field, kappa0: float, half_power: int, mean: int = MEAN_ARITHMETIC,
                                     rho=None, inv_dt: float = 1.0, stream=None):
        """maspcg_set_coefficients_from_fields: kappa = kappa0 field^(half_power/2) on faces, s = inv_dt rho."""
        self._check(self._L.maspcg_set_coefficients_from_fields(self.ctx, _ptr(field), float(kappa0), int(half_power),
                                                                int(mean), _ptr(rho), float(inv_dt), _stream(stream)))

    def set_bc_r(self, bc_in: int, g_in, bc_out: int, g_out, stream=None):
        host = isinstance(g_in, np.ndarray) or isinstance(g_out, np.ndarray) or (g_in is None and g_out is None)
        fn = self._L.maspcg_set_bc_r_host if host else self._L.maspcg_set_bc_r
        self._check(fn(self.ctx, int(bc_in), _ptr(g_in), int(bc_out), _ptr(g_out), _stream(stream)))

    def solve(self, rhs, x, tol: float, maxit: int, stream=None, raise_on_error: bool = True):
        """maspcg_solve (device tensors) / maspcg_solve_host (numpy arrays; x updated in place).
        Returns (status, info_dict, hist ndarray[iters+1])."""
        host = isinstance(x, np.ndarray)
        fn = self._L.maspcg_solve_host if host else self._L.maspcg_solve
        hist = np.zeros(maxit + 1)
        info = Info()
        st = fn(self.ctx, _ptr(rhs), _ptr(x), float(tol), int(maxit), hist.ctypes.data, ctypes.byref(info),
                _stream(stream))
        if raise_on_error and st < 0:
            self._check(st)
        d = {"iters": info.iters, "bnorm": info.bnorm, "rnorm": info.rnorm, "rel_resid": info.rel_resid}
        if st < 0:
            d["error"] = (self._L.maspcg_last_error(self.ctx) or b"").decode()
        return st, d, hist[: max(info.iters, 0) + 1].copy()

    def apply(self, x, y=None, stream=None):
        import torch
        if y is None:
            y = torch.empty_like(x)
        self._check(self._L.maspcg_apply(self.ctx, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def sts_step(self, u, tau: float, stages: int, stream=None):
        """maspcg_sts_step: one RKL2 super-time-step of V du/dt = b_D - K u, in place on u."""
        self._check(self._L.maspcg_sts_step(self.ctx, _ptr(u), float(tau), int(stages), _stream(stream)))
        return u

    def sts_dt_limit(self, stream=None) -> float:
        """maspcg_sts_dt_limit: the forward-Euler step bound 2 / max_c (K_cc + sum T)/V_c."""
        v = ctypes.c_double()
        self._check(self._L.maspcg_sts_dt_limit(self.ctx, ctypes.byref(v), _stream(stream)))
        return v.value

    def get_operator(self, stream=None):
        nloc, nt, nr = self.local_shape
        Tr = np.empty((nloc, nt, nr + 1))
        Tt = np.empty((nloc, nt + 1, nr))
        Tp = np.empty((nloc, nt, nr))
        D = np.empty((nloc, nt, nr))
        self._check(self._L.maspcg_get_operator(self.ctx, _ptr(Tr), _ptr(Tt), _ptr(Tp), _ptr(D),
                                                _stream(stream)))
        return Tr, Tt, Tp, D

    # ---------------------------------------------------------------- field-aligned conduction (NEXT-4)
    def aniso_enable(self):
        """Allocate and attach the cross terms' workspace (maspcg_aniso_workspace_bytes / _set_workspace)."""
        import torch
        if getattr(self, "aniso_workspace", None) is not None:
            return
        nbytes = self._L.maspcg_aniso_workspace_bytes(self.ctx)
        self.aniso_workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        base = self.aniso_workspace.data_ptr()
        self._check(self._L.maspcg_aniso_set_workspace(self.ctx, base + (-base) % 256, nbytes))

    def set_aniso_coefficients(self, krt, krp, ktp, stream=None):
        """maspcg_set_aniso_coefficients: edge cross coefficients kappa_par b_a b_b (device tensors
        [nloc][nt+1][nr+1], [nloc][nt][nr+1], [nloc][nt+1][nr]); all None: back to the 7-point operator."""
        self.aniso_enable()
        self._check(self._L.maspcg_set_aniso_coefficients(self.ctx, _ptr(krt), _ptr(krp), _ptr(ktp), _stream(stream)))

    def aniso_get_operator(self, stream=None):
        """maspcg_aniso_get_operator: (Xrt, Xrp, Xtp, D7) in the library layout [nloc][nt][nr] (host copies)."""
        out = [np.empty(self.local_shape) for _ in range(4)]
        self._check(self._L.maspcg_aniso_get_operator(self.ctx, *(_ptr(a) for a in out), _stream(stream)))
        return tuple(out)

    # ---------------------------------------------------------------- vector viscosity (NEXT-2)
    @property
    def vv_local_shape(self):
        return (self.nloc, 3, self.nt, self.nr)

    def vv_enable(self):
        """Allocate and attach the vector operator's workspace (maspcg_vv_workspace_bytes / _set_workspace)."""
        import torch
        if getattr(self, "vv_workspace", None) is not None:
            return
        nbytes = self._L.maspcg_vv_workspace_bytes(self.ctx)
        self.vv_workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        base = self.vv_workspace.data_ptr()
        self._check(self._L.maspcg_vv_set_workspace(self.ctx, base + (-base) % 256, nbytes))
        if getattr(self, "_ipc", False):
            self._peer_exchange(1)

    def vv_set_coefficients(self, nu, s, stream=None):
        """maspcg_vv_set_coefficients: cell viscosity and shift, device [nloc][nt][nr]."""
        self.vv_enable()
        self._check(self._L.maspcg_vv_set_coefficients(self.ctx, _ptr(nu), _ptr(s), _stream(stream)))

    def vv_set_bc_r(self, wall_in: int, g_in, wall_out: int, g_out, stream=None):
        """maspcg_vv_set_bc_r: wall types and wall data, device [nloc][3][nt] or None."""
        self.vv_enable()
        self._check(self._L.maspcg_vv_set_bc_r(self.ctx, int(wall_in), _ptr(g_in), int(wall_out), _ptr(g_out),
                                               _stream(stream)))

    def vv_apply(self, x, y=None, stream=None):
        import torch
        if y is None:
            y = torch.empty_like(x)
        self._check(self._L.maspcg_vv_apply(self.ctx, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def vv_solve(self, f, x, tol: float, maxit: int, stream=None, raise_on_error: bool = True):
        """maspcg_vv_solve (device [nloc][3][nt][nr]); returns (status, info_dict, hist)."""
        hist = np.zeros(maxit + 1)
        info = Info()
        st = self._L.maspcg_vv_solve(self.ctx, _ptr(f), _ptr(x), float(tol), int(maxit), hist.ctypes.data,
                                     ctypes.byref(info), _stream(stream))
        if raise_on_error and st < 0:
            self._check(st)
        d = {"iters": info.iters, "bnorm": info.bnorm, "rnorm": info.rnorm, "rel_resid": info.rel_resid}
        if st < 0:
            d["error"] = (self._L.maspcg_last_error(self.ctx) or b"").decode()
        return st, d, hist[: max(info.iters, 0) + 1].copy()

    def vv_get_diag(self, stream=None) -> np.ndarray:
        D = np.empty(self.vv_local_shape)
        self._check(self._L.maspcg_vv_get_diag(self.ctx, _ptr(D), _stream(stream)))
        return D

    def stats(self) -> dict:
        s = Stats()
        self._check(self._L.maspcg_get_stats(self.ctx, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        self._check(self._L.maspcg_reset_stats(self.ctx))


class LoopbackGroup:
    """In-process multi-rank emulation on one device (maspcg_loopback_group_create; TEST ONLY):
    one Solver(..., loopback=(group, rank)) per rank, each driven from its own host thread."""

    def __init__(self, nranks: int):
        self._L = lib()
        h = ctypes.c_void_p()
        st = self._L.maspcg_loopback_group_create(nranks, ctypes.byref(h))
        if st != OK:
            raise MaspcgError(st, self._L.maspcg_last_error(None).decode())
        self.handle, self.nranks = h, nranks

    def close(self):
        if self.handle:
            self._L.maspcg_loopback_group_destroy(self.handle)
            self.handle = None


def solver_for_problem(prob, *, group=None, device=None, chunk=16, stream=None, loopback=None, force_comm=False,
                       comm="nccl"):
    """Create a Solver for an inputs.Problem slab and upload its coefficients and BCs (device copies)."""
    import torch
    dev = f"cuda:{torch.cuda.current_device() if device is None else device}"
    S = Solver(prob.nr, prob.nt, prob.np, prob.rf, prob.tf, prob.pf, group=group, device=device, chunk=chunk,
               loopback=loopback, force_comm=force_comm, comm=comm)
    assert (S.k0, S.nloc) == (prob.k0, prob.nloc), "problem slab does not match the library's decomposition"
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    S.set_coefficients(T(prob.kr), T(prob.kt), T(prob.kp), T(prob.s), stream)
    S.set_bc_r(prob.bc_in, T(prob.g_in), prob.bc_out, T(prob.g_out), stream) if (
        prob.g_in is not None or prob.g_out is not None) else S.set_bc_r(prob.bc_in, None, prob.bc_out, None,
                                                                           stream)
    if getattr(prob, "krt", None) is not None:   # field-aligned conduction (inputs.AnisoProblem)
        S.set_aniso_coefficients(T(prob.krt), T(prob.krp), T(prob.ktp), stream)
    return S
