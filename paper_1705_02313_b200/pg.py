"""Thin ctypes binding of ``libpgsi.so`` (C ABI in ``include/pg.h``).

Argument marshalling only: every step of the path (valuation, switches, loop
control, ABI-order exports) runs in the library's CUDA kernels. There is no CPU
fallback: if the shared library is missing or CUDA is unavailable the calls
raise. Host arrays are numpy; in device-pointer mode (``device_ptrs=True``)
strategy/val/top/winner buffers are torch CUDA tensors (PyTorch is used only for
device memory and streams).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpgsi.so")

PG_SINK = -1
PG_NONE = -2
PG_NO_PREPROCESS = 1
PG_CHECK_INVARIANTS = 2
PG_PHASE_TIMING = 4
PG_PTRS_ON_DEVICE = 8
PG_NO_INCREMENTAL = 16
PG_HOST_LOAD = 32
PG_BFS = 64
PG_SI_RESET = 128
PG_BELLMAN_FORD = 256
PG_TRACE = 512
BEST_RESPONSE = {"si": 0, "si_reset": PG_SI_RESET, "bf": PG_BELLMAN_FORD}

STATUS = {0: "PG_OK", -1: "PG_EINVAL", -2: "PG_ENOMEM", -3: "PG_ECUDA", -4: "PG_ENCCL",
          -5: "PG_EINADMISSIBLE", -6: "PG_EITERCAP", -7: "PG_ESTATE", -8: "PG_ENOTSUP"}


class PGError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"{self.name}: {msg}")


class Options(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("device", C.c_int32), ("stream", C.c_void_p),
                ("splitter_k", C.c_int32), ("prefix_pairs", C.c_int32),
                ("max_inner", C.c_int64), ("max_outer", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "n", "n_internal", "m", "m_internal", "d", "dummies", "inner_iters", "outer_passes",
        "odd_switches", "even_switches", "v1_rounds", "v2_split_valuations", "max_depth",
        "gpu_launches")] + [(k, C.c_double) for k in (
            "ms_load", "ms_call", "ms_v1", "ms_v2", "ms_odd", "ms_even", "ms_other")] + [
        (k, C.c_int64) for k in ("n_v1", "n_v2", "n_odd", "n_even")] + [
        (k, C.c_double) for k in ("bytes_v1", "bytes_v2", "bytes_odd", "bytes_even")] + [
        ("full_compares", C.c_int64), ("walk_steps", C.c_int64), ("top_vertices", C.c_int64),
        ("inc_valuations", C.c_int64), ("inc_even_switches", C.c_int64), ("inc_aborts", C.c_int64),
        ("bfs_valuations", C.c_int64), ("bfs_aborts", C.c_int64), ("ms_bfs", C.c_double),
        ("n_bfs", C.c_int64), ("bytes_bfs", C.c_double),
        ("dirty_vertices", C.c_int64),
        ("ms_inc", C.c_double),
        ("n_inc", C.c_int64), ("bytes_inc", C.c_double),
        ("dist_exchanges", C.c_int64), ("dist_bytes", C.c_int64), ("ms_dist", C.c_double),
        ("prefix_gathers", C.c_int64), ("small_solves", C.c_int64),
        ("bf_rounds", C.c_int64), ("ms_bf", C.c_double), ("n_bf", C.c_int64),
        ("device_loop_solves", C.c_int64), ("bytes_bf", C.c_double), ("cluster_solves", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# int (*)(void *ctx, const void *send, void *recv, int64_t bytes, int32_t on_device)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libpgsi.so (raises if absent: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P = C.c_void_p
    L.pg_load.argtypes = [C.c_int64, P, P, P, P, C.POINTER(Options), C.POINTER(C.c_void_p)]
    L.pg_info.argtypes = [C.c_void_p, P, P, P, P]
    L.pg_valuate.argtypes = [C.c_void_p, P, P, P, P]
    L.pg_best_response.argtypes = [C.c_void_p, P, P, P, P, P, P]
    L.pg_solve.argtypes = [C.c_void_p, P, P, P, P, C.POINTER(Stats)]
    L.pg_get_stats.argtypes = [C.c_void_p, C.POINTER(Stats)]
    L.pg_get_trace.argtypes = [C.c_void_p, P, C.c_int64, P]
    L.pg_dist_unique_id.argtypes = [P, C.c_int64]
    L.pg_dist_init.argtypes = [C.c_void_p, P, C.c_int32, C.c_int32]
    L.pg_inspect.argtypes = [C.c_int64, P, P, P, P, C.c_uint32] + [P] * 9
    L.pg_dist_attach.argtypes = [C.c_void_p, C.c_int32, C.c_int32, ALLGATHER_FN, P]
    for f in ("pg_load", "pg_info", "pg_valuate", "pg_best_response", "pg_solve", "pg_get_stats",
              "pg_inspect", "pg_dist_attach", "pg_get_trace", "pg_dist_unique_id", "pg_dist_init"):
        getattr(L, f).restype = C.c_int
    L.pg_parse_pgsolver.argtypes = [C.c_char_p, C.c_int64, P, P, P, P, P, P]
    L.pg_format_solution.argtypes = [C.c_int64, P, P, P, P, C.c_char_p, C.c_int64, P]
    L.pg_verify_solution.argtypes = [C.c_int64, P, P, P, P, P, P, P, P]
    L.pg_verify_solution_device.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_int32, P, P]
    for f in ("pg_parse_pgsolver", "pg_format_solution", "pg_verify_solution", "pg_verify_solution_device"):
        getattr(L, f).restype = C.c_int
    L.pg_free.argtypes = [C.c_void_p]
    L.pg_free.restype = None
    L.pg_last_error.restype = C.c_char_p
    L.pg_version.restype = C.c_char_p
    _lib = L
    return L


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())  # torch tensor


@dataclass
class SolveResult:
    winner: object
    sigma: object
    tau: object
    val: object
    stats: dict


class Game:
    """A game loaded on the GPU (``pg_load``)."""

    def __init__(self, n, row_ptr, col, owner, priority, *, device: int = 0, stream=None,
                 preprocess: bool = True, check: bool = False, phase_timing: bool = False,
                 device_ptrs: bool = False, splitter_k: int = 0, max_inner: int = 0,
                 max_outer: int = 0, prefix_pairs: int = 0, incremental: bool = True,
                 host_load: bool = False, bfs: bool = False, best_response: str = "si",
                 trace: bool = False):
        """best_response: "si" (Algorithm 1), "si_reset" (PG_SI_RESET) or "bf"
        (PG_BELLMAN_FORD), the arms of the paper's Table 2.
        trace: record the per-iteration parity trace (PG_TRACE; ``get_trace``)."""
        L = load_library()
        self._in = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                    np.ascontiguousarray(owner, np.uint8), np.ascontiguousarray(priority, np.int32))
        flags = ((0 if preprocess else PG_NO_PREPROCESS) | (PG_CHECK_INVARIANTS if check else 0) |
                 (PG_PHASE_TIMING if phase_timing else 0) | (PG_PTRS_ON_DEVICE if device_ptrs else 0) |
                 (0 if incremental else PG_NO_INCREMENTAL) | (PG_HOST_LOAD if host_load else 0) |
                 (PG_BFS if bfs else 0) | BEST_RESPONSE[best_response] | (PG_TRACE if trace else 0))
        opt = Options(flags, device, C.c_void_p(stream) if stream else None, splitter_k,
                      prefix_pairs, max_inner, max_outer)
        h = C.c_void_p()
        rc = L.pg_load(int(n), *[_ptr(a) for a in self._in], C.byref(opt), C.byref(h))
        self._in = None
        if rc:
            raise PGError(rc, L.pg_last_error().decode())
        self._h = h
        self.device = device
        self.device_ptrs = device_ptrs
        self.n = int(n)
        ni = C.c_int64()
        d = C.c_int32()
        du = C.c_int64()
        L.pg_info(h, C.byref(ni), C.byref(d), None, C.byref(du))
        self.n_internal, self.d, self.dummies = ni.value, d.value, du.value
        self.priorities = np.zeros(self.d, np.int32)
        L.pg_info(h, None, None, _ptr(self.priorities), None)

    @classmethod
    def from_game(cls, g, **kw):
        return cls(g.n, g.row_ptr, g.col, g.owner, g.priority, **kw)

    def _check(self, rc):
        if rc:
            raise PGError(rc, _lib.pg_last_error().decode())

    def free(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.pg_free(self._h)
            self._h = None

    __del__ = free

    def _alloc(self, shape, dtype):
        if self.device_ptrs:
            import torch
            tdt = {np.int32: torch.int32, np.uint8: torch.uint8}[dtype]
            return torch.empty(shape, dtype=tdt, device=f"cuda:{self.device}")
        return np.empty(shape, dtype)

    def _arg(self, a, dtype):
        if a is None:
            return None
        if self.device_ptrs:
            return a
        return np.ascontiguousarray(a, dtype)

    def attach_dist(self, rank: int, world: int, allgather=None):
        """Make this handle rank `rank` of `world` ranks solving the same game with
        range-sharded switch steps (``pg_dist_attach``).
        ``allgather(send_ptr, recv_ptr, nbytes, on_device)`` must gather nbytes from
        every rank into recv (rank order) and return when done, raising on failure
        (see ``paper_1705_02313_b200.dist.torch_allgather``). world = 1 detaches."""
        if allgather is None or world == 1:
            self._dist_cb = None
            self._check(_lib.pg_dist_attach(self._h, int(rank), int(world), ALLGATHER_FN(), None))
            return

        def cb(_ctx, send, recv, nbytes, on_device):
            try:
                allgather(int(send or 0), int(recv or 0), int(nbytes), bool(on_device))
                return 0
            except BaseException as e:   # noqa: BLE001 - reported through the C status
                self.dist_error = e
                return 1

        self._dist_cb = ALLGATHER_FN(cb)   # keep the trampoline alive with the handle
        self.dist_error = None
        self._check(_lib.pg_dist_attach(self._h, int(rank), int(world), self._dist_cb, None))

    def dist_init(self, nccl_id: bytes, rank: int, world: int):
        """Join `world` ranks solving this same game with the library's own NCCL
        communicator (``pg_dist_init``); ``nccl_id`` from :func:`dist_unique_id` on rank 0."""
        buf = C.create_string_buffer(bytes(nccl_id), len(nccl_id))
        self._check(_lib.pg_dist_init(self._h, buf, int(rank), int(world)))

    def stats(self) -> dict:
        s = Stats()
        self._check(_lib.pg_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def get_trace(self) -> np.ndarray:
        """Per-iteration parity trace of the last solve / best response (``pg_get_trace``):
        uint64 [records, 5] rows (kind, h_succ, h_val, n_top, switches)."""
        n = C.c_int64()
        self._check(_lib.pg_get_trace(self._h, None, 0, C.byref(n)))
        rec = np.zeros((max(n.value, 1), 5), np.uint64)
        self._check(_lib.pg_get_trace(self._h, _ptr(rec), n.value, C.byref(n)))
        return rec[:n.value]

    def valuate(self, strategy, want_cycle_dom: bool = True):
        N, d = self.n_internal, self.d
        s = self._arg(strategy, np.int32)
        val = self._alloc((N, d), np.int32)
        top = self._alloc((N,), np.uint8)
        cd = self._alloc((N,), np.int32) if want_cycle_dom else None
        self._check(_lib.pg_valuate(self._h, _ptr(s), _ptr(val), _ptr(top), _ptr(cd)))
        return val, top, cd

    def best_response(self, sigma, tau0=None):
        N, d = self.n_internal, self.d
        s = self._arg(sigma, np.int32)
        t0 = self._arg(tau0, np.int32)
        tau = self._alloc((N,), np.int32)
        val = self._alloc((N, d), np.int32)
        top = self._alloc((N,), np.uint8)
        inner = C.c_int64()
        self._check(_lib.pg_best_response(self._h, _ptr(s), _ptr(t0), _ptr(tau), _ptr(val),
                                          _ptr(top), C.byref(inner)))
        return tau, val, top, inner.value

    def solve(self, want_strategies: bool = True, want_val: bool = False, out=None) -> SolveResult:
        """``out`` may supply preallocated (winner, sigma, tau, val) buffers."""
        n, d = self.n, self.d
        if out is not None:
            winner, sigma, tau, val = out
        else:
            winner = self._alloc((n,), np.uint8)
            sigma = self._alloc((n,), np.int32) if want_strategies else None
            tau = self._alloc((n,), np.int32) if want_strategies else None
            val = self._alloc((n, d), np.int32) if want_val else None
        st = Stats()
        self._check(_lib.pg_solve(self._h, _ptr(winner), _ptr(sigma), _ptr(tau), _ptr(val),
                                  C.byref(st)))
        return SolveResult(winner, sigma, tau, val, st.as_dict())


def inspect(g, preprocess: bool = True):
    """Host-side load transform only (no GPU): returns dict with the internal game
    in ABI order (owner, pidx, adj_ptr, adj, priorities, dummies)."""
    L = load_library()
    arrs = (np.ascontiguousarray(g.row_ptr, np.int64), np.ascontiguousarray(g.col, np.int32),
            np.ascontiguousarray(g.owner, np.uint8), np.ascontiguousarray(g.priority, np.int32))
    flags = 0 if preprocess else PG_NO_PREPROCESS
    ni, d, du, mi = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64()
    rc = L.pg_inspect(g.n, *[_ptr(a) for a in arrs], flags, C.byref(ni), C.byref(d), C.byref(du),
                      C.byref(mi), None, None, None, None, None)
    if rc:
        raise PGError(rc, L.pg_last_error().decode())
    owner = np.zeros(ni.value, np.uint8)
    pidx = np.zeros(ni.value, np.int32)
    adj_ptr = np.zeros(ni.value + 1, np.int64)
    adj = np.zeros(max(mi.value, 1), np.int32)
    pri = np.zeros(max(d.value, 1), np.int32)
    rc = L.pg_inspect(g.n, *[_ptr(a) for a in arrs], flags, None, None, None, None, _ptr(owner),
                      _ptr(pidx), _ptr(adj_ptr), _ptr(adj), _ptr(pri))
    if rc:
        raise PGError(rc, L.pg_last_error().decode())
    return dict(n_internal=ni.value, d=d.value, dummies=du.value, owner=owner, pidx=pidx,
                adj_ptr=adj_ptr, adj=adj[:mi.value], priorities=pri[:d.value])


def dist_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for :meth:`Game.dist_init` (``pg_dist_unique_id``)."""
    L = load_library()
    buf = C.create_string_buffer(128)
    rc = L.pg_dist_unique_id(buf, 128)
    if rc:
        raise PGError(rc, L.pg_last_error().decode())
    return buf.raw


def version() -> str:
    return load_library().pg_version().decode()


@dataclass
class ParsedGame:
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    owner: np.ndarray
    priority: np.ndarray

    @property
    def m(self):
        return int(self.row_ptr[-1])


def parse_pgsolver(text) -> ParsedGame:
    """PGSolver text -> CSR game (``pg_parse_pgsolver``, host C++)."""
    L = load_library()
    b = text.encode() if isinstance(text, str) else bytes(text)
    n, m = C.c_int64(), C.c_int64()
    rc = L.pg_parse_pgsolver(b, len(b), C.byref(n), C.byref(m), None, None, None, None)
    if rc:
        raise PGError(rc, L.pg_last_error().decode())
    rp = np.zeros(n.value + 1, np.int64)
    col = np.zeros(max(m.value, 1), np.int32)
    own = np.zeros(max(n.value, 1), np.uint8)
    pri = np.zeros(max(n.value, 1), np.int32)
    rc = L.pg_parse_pgsolver(b, len(b), None, None, _ptr(rp), _ptr(col), _ptr(own), _ptr(pri))
    if rc:
        raise PGError(rc, L.pg_last_error().decode())
    return ParsedGame(n.value, rp, col[:m.value], own[:n.value], pri[:n.value])


def format_solution(owner, winner, sigma, tau) -> str:
    """PGSolver solution text (``pg_format_solution``)."""
    L = load_library()
    arrs = [np.ascontiguousarray(owner, np.uint8), np.ascontiguousarray(winner, np.uint8),
            np.ascontiguousarray(sigma, np.int32), np.ascontiguousarray(tau, np.int32)]
    n = len(arrs[0])
    ln = C.c_int64()
    rc = L.pg_format_solution(n, *[_ptr(a) for a in arrs], None, 0, C.byref(ln))
    if rc:
        raise PGError(rc, L.pg_last_error().decode())
    buf = C.create_string_buffer(ln.value + 1)
    rc = L.pg_format_solution(n, *[_ptr(a) for a in arrs], buf, ln.value + 1, C.byref(ln))
    if rc:
        raise PGError(rc, L.pg_last_error().decode())
    return buf.value.decode()


def verify_solution(g, winner, sigma, tau, device=None):
    """(ok, witness, message) from ``pg_verify_solution`` on the original game g
    (host C++), or from ``pg_verify_solution_device`` on GPU ``device``."""
    L = load_library()
    arrs = [np.ascontiguousarray(g.row_ptr, np.int64), np.ascontiguousarray(g.col, np.int32),
            np.ascontiguousarray(g.owner, np.uint8), np.ascontiguousarray(g.priority, np.int32),
            np.ascontiguousarray(winner, np.uint8), np.ascontiguousarray(sigma, np.int32),
            np.ascontiguousarray(tau, np.int32)]
    w = C.c_int64()
    if device is not None:
        rounds = C.c_int64()
        rc = L.pg_verify_solution_device(int(g.n), *[_ptr(a) for a in arrs], int(device), C.byref(w),
                                         C.byref(rounds))
    else:
        rc = L.pg_verify_solution(int(g.n), *[_ptr(a) for a in arrs], C.byref(w))
    if rc == 0:
        return True, -1, ""
    if rc != -1:
        raise PGError(rc, L.pg_last_error().decode())
    return False, w.value, L.pg_last_error().decode()

