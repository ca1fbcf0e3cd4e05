"""ctypes wrapper around ``liboracle.so`` (TEST INFRASTRUCTURE ONLY; see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_CODES = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -5: "EINADMISSIBLE", -6: "EITERCAP"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle {OR_CODES.get(code, code)}: {msg}")
        self.code = code
        self.name = OR_CODES.get(code, str(code))


def oracle_lib_path() -> str:
    return _LIB


def build_oracle(force: bool = False) -> str:
    """Compile the plain C oracle (gcc -O2, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        L.oracle_load.argtypes = [C.c_int64, P, P, P, P, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_load.restype = C.c_int
        L.oracle_free.argtypes = [C.c_void_p]
        L.oracle_last_error.restype = C.c_char_p
        for f in ("oracle_n_internal", "oracle_dummies", "oracle_m_internal"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_int64
        L.oracle_d.argtypes = [C.c_void_p]
        L.oracle_d.restype = C.c_int32
        L.oracle_priorities.argtypes = [C.c_void_p, P]
        L.oracle_export.argtypes = [C.c_void_p, P, P, P, P, P]
        L.oracle_valuate.argtypes = [C.c_void_p, P, P, P, P]
        L.oracle_valuate.restype = C.c_int
        L.oracle_best_response.argtypes = [C.c_void_p, P, P, P, P, P, P]
        L.oracle_best_response.restype = C.c_int
        L.oracle_solve.argtypes = [C.c_void_p, C.c_int64, C.c_int64, P, P, P, P, P, P, P, P,
                                   P, C.c_int64, P, C.c_int64]
        L.oracle_solve.restype = C.c_int
        L.oracle_solve_mode.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, P, P, P, P, P, P,
                                        P, P, P, C.c_int64, P, C.c_int64]
        L.oracle_solve_mode.restype = C.c_int
        L.oracle_solve_traced.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, P, P, P, P, P, P,
                                          P, P, P, C.c_int64, P]
        L.oracle_solve_traced.restype = C.c_int
        L.oracle_best_response_bf.argtypes = [C.c_void_p, P, P, P, P, P]
        L.oracle_best_response_bf.restype = C.c_int
        L.oracle_switch_step.argtypes = [C.c_void_p, P, C.c_int, P, P]
        L.oracle_switch_step.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class SolveResult:
    winner: np.ndarray
    sigma: np.ndarray
    tau: np.ndarray
    val: np.ndarray
    succ_int: np.ndarray
    val_int: np.ndarray
    top_int: np.ndarray
    inner_iters: int
    outer_passes: int
    odd_trace: np.ndarray
    even_trace: np.ndarray
    trace: np.ndarray | None = None   # per-iteration parity trace, uint64 [records, 5]


class Oracle:
    """A loaded (canonicalised + preprocessed) game inside the oracle."""

    def __init__(self, game, preprocess: bool = True):
        L = _load()
        self._keep = (np.ascontiguousarray(game.row_ptr, np.int64),
                      np.ascontiguousarray(game.col, np.int32),
                      np.ascontiguousarray(game.owner, np.uint8),
                      np.ascontiguousarray(game.priority, np.int32))
        h = C.c_void_p()
        rc = L.oracle_load(game.n, *[_p(a) for a in self._keep], int(preprocess), C.byref(h))
        if rc:
            raise OracleError(rc, L.oracle_last_error().decode())
        self._h = h
        self.n = game.n
        self.n_internal = L.oracle_n_internal(h)
        self.d = L.oracle_d(h)
        self.dummies = L.oracle_dummies(h)
        self.priorities = np.zeros(self.d, np.int32)
        L.oracle_priorities(h, _p(self.priorities))

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.oracle_free(self._h)
            self._h = None

    def internal(self):
        """(owner, pidx, adj_ptr, adj, dummy_of) of the preprocessed game."""
        L = _load()
        N = self.n_internal
        owner = np.zeros(N, np.uint8)
        pidx = np.zeros(N, np.int32)
        adj_ptr = np.zeros(N + 1, np.int64)
        adj = np.zeros(max(L.oracle_m_internal(self._h), 1), np.int32)
        dummy_of = np.zeros(max(self.dummies, 1), np.int64)
        L.oracle_export(self._h, _p(owner), _p(pidx), _p(adj_ptr), _p(adj), _p(dummy_of))
        return owner, pidx, adj_ptr, adj[:adj_ptr[-1]], dummy_of[:self.dummies]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, _load().oracle_last_error().decode())

    def valuate(self, strategy):
        N, d = self.n_internal, self.d
        s = np.ascontiguousarray(strategy, np.int32)
        val = np.zeros((N, d), np.int32)
        top = np.zeros(N, np.uint8)
        cdom = np.zeros(N, np.int32)
        self._check(_load().oracle_valuate(self._h, _p(s), _p(val), _p(top), _p(cdom)))
        return val, top, cdom

    def best_response(self, sigma, tau0=None):
        N, d = self.n_internal, self.d
        s = np.ascontiguousarray(sigma, np.int32)
        t0 = None if tau0 is None else np.ascontiguousarray(tau0, np.int32)
        tau = np.zeros(N, np.int32)
        val = np.zeros((N, d), np.int32)
        top = np.zeros(N, np.uint8)
        inner = np.zeros(1, np.int64)
        self._check(_load().oracle_best_response(self._h, _p(s), _p(t0), _p(tau), _p(val),
                                                  _p(top), _p(inner)))
        return tau, val, top, int(inner[0])

    MODES = {"si": 0, "si_reset": 1, "bf": 2}

    def best_response_bf(self, sigma):
        """Bellman-Ford best response: (τ, val, top, rounds)."""
        N, d = self.n_internal, self.d
        s = np.ascontiguousarray(sigma, np.int32)
        tau = np.zeros(N, np.int32)
        val = np.zeros((N, d), np.int32)
        top = np.zeros(N, np.uint8)
        rounds = np.zeros(1, np.int64)
        self._check(_load().oracle_best_response_bf(self._h, _p(s), _p(tau), _p(val), _p(top),
                                                     _p(rounds)))
        return tau, val, top, int(rounds[0])

    def solve(self, max_inner: int = 0, max_outer: int = 0, trace_cap: int = 1 << 16,
              mode: str = "si") -> SolveResult:
        """Algorithm 1; mode "si" (warm-started τ), "si_reset" (τ := τ_init before every
        best response) or "bf" (Bellman-Ford best responses; inner_iters
        counts relaxation rounds)."""
        n, N, d = self.n, self.n_internal, self.d
        winner = np.zeros(n, np.uint8)
        sigma = np.zeros(n, np.int32)
        tau = np.zeros(n, np.int32)
        val = np.zeros((n, d), np.int32)
        succ_int = np.zeros(N, np.int32)
        val_int = np.zeros((N, d), np.int32)
        top_int = np.zeros(N, np.uint8)
        stats = np.zeros(8, np.int64)
        ot = np.zeros(trace_cap, np.int64)
        et = np.zeros(trace_cap, np.int64)
        self._check(_load().oracle_solve_mode(self._h, self.MODES[mode], max_inner, max_outer,
                                              _p(winner), _p(sigma),
                                         _p(tau), _p(val), _p(succ_int), _p(val_int), _p(top_int),
                                         _p(stats), _p(ot), trace_cap, _p(et), trace_cap))
        inner, outer = int(stats[0]), int(stats[1])
        return SolveResult(winner, sigma, tau, val, succ_int, val_int, top_int, inner, outer,
                           ot[:min(inner, trace_cap)].copy(), et[:min(outer, trace_cap)].copy())

    def solve_traced(self, max_inner: int = 0, max_outer: int = 0, mode: str = "si",
                     cap: int = 1 << 16) -> SolveResult:
        """solve() plus the per-iteration parity trace: one record
        (0, h_succ, h_val, n_top, odd switches) per valuation and (1, 0, 0, 0, even
        switches) per All_Even step, as uint64 [records, 5]."""
        n, N, d = self.n, self.n_internal, self.d
        winner = np.zeros(n, np.uint8)
        sigma = np.zeros(n, np.int32)
        tau = np.zeros(n, np.int32)
        val = np.zeros((n, d), np.int32)
        succ_int = np.zeros(N, np.int32)
        top_int = np.zeros(N, np.uint8)
        stats = np.zeros(8, np.int64)
        tr = np.zeros((cap, 5), np.uint64)
        tl = np.zeros(1, np.int64)
        self._check(_load().oracle_solve_traced(self._h, self.MODES[mode], max_inner, max_outer, _p(winner),
                                                _p(sigma), _p(tau), _p(val), _p(succ_int), None,
                                                _p(top_int), _p(stats), _p(tr), cap, _p(tl)))
        inner, outer = int(stats[0]), int(stats[1])
        return SolveResult(winner, sigma, tau, val, succ_int, None, top_int, inner, outer,
                           np.zeros(0, np.int64), np.zeros(0, np.int64), tr[:min(int(tl[0]), cap)].copy())

    def switch_step(self, succ, side: int):
        out = np.zeros(self.n_internal, np.int32)
        cnt = np.zeros(1, np.int64)
        s = np.ascontiguousarray(succ, np.int32)
        self._check(_load().oracle_switch_step(self._h, _p(s), side, _p(out), _p(cnt)))
        return out, int(cnt[0])
