"""ctypes front-end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package.  The product path (paper_2403_16125_b200) never
does, and shares no code with it; both only consume the seeded arrays of
paper_2403_16125_b200.workload.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libcrius_oracle.so")
SRC = os.path.join(HERE, "crius_oracle.cpp")
INF = np.iinfo(np.int64).max


def build(force=False):
    """g++ -O2, single thread, no FMA contraction, no fast-math."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "crius_oracle.h"))):
        return LIB
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
                           "-shared", "-fPIC", "-o", LIB, SRC])
    return LIB


class _Problem(C.Structure):
    _fields_ = [
        ("n_types", C.c_int32), ("cap", C.c_void_p), ("gpn", C.c_void_p), ("mem", C.c_void_p),
        ("alpha_in", C.c_void_p), ("beta_in", C.c_void_p), ("alpha_x", C.c_void_p),
        ("beta_x", C.c_void_p), ("n_jobs", C.c_int32), ("k_max", C.c_int32),
        ("job_id", C.c_void_p), ("submit", C.c_void_p), ("ng", C.c_void_p), ("gb", C.c_void_p),
        ("kst", C.c_void_p), ("n_layers", C.c_void_p), ("layer_off", C.c_void_p),
        ("c", C.c_void_p), ("w", C.c_void_p), ("act", C.c_void_p), ("bnd", C.c_void_p),
        ("tpv", C.c_void_p), ("tpn", C.c_void_p), ("gpu_set", C.c_int32), ("s_max", C.c_int32),
        ("g_max", C.c_int32), ("b_mode", C.c_int32), ("b_count", C.c_int32),
        ("b_values", C.c_void_p), ("depth", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_comm.restype = C.c_int64
        _lib.oracle_comm.argtypes = [C.c_int32] + [C.c_int64] * 5
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Holds a Problem's arrays (kept alive) and the ctypes struct."""

    def __init__(self, pr):
        self.pr = pr
        keep = {}

        def arr(name, dtype):
            a = np.ascontiguousarray(getattr(pr, name), dtype=dtype)
            keep[name] = a
            return _ptr(a)

        bv = np.ascontiguousarray(pr.b_values, np.int32)
        if bv.size == 0:
            bv = np.zeros(1, np.int32)
        keep["b_values"] = bv
        self._keep = keep
        self.s = _Problem(
            n_types=pr.n_types, cap=arr("cap", np.int32), gpn=arr("gpn", np.int32),
            mem=arr("mem", np.int64), alpha_in=arr("alpha_in", np.int64),
            beta_in=arr("beta_in", np.int64), alpha_x=arr("alpha_x", np.int64),
            beta_x=arr("beta_x", np.int64), n_jobs=pr.n_jobs, k_max=pr.k_max,
            job_id=arr("job_id", np.int64), submit=arr("submit", np.int64), ng=arr("ng", np.int32),
            gb=arr("gb", np.int32), kst=arr("kst", np.int32), n_layers=arr("n_layers", np.int32),
            layer_off=arr("layer_off", np.int64), c=arr("c", np.int32), w=arr("w", np.int64),
            act=arr("act", np.int64), bnd=arr("bnd", np.int64), tpv=arr("tpv", np.int64),
            tpn=arr("tpn", np.int32), gpu_set=pr.gpu_set, s_max=pr.s_max, g_max=pr.g_max,
            b_mode=pr.b_mode, b_count=int(pr.b_values.size) if pr.b_mode == 1 else 0,
            b_values=_ptr(bv), depth=pr.depth)
        self.L = lib()

    def _check(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"oracle {what} failed with code {rc}")

    def count(self):
        n, p = C.c_int64(), C.c_int64()
        self._check(self.L.oracle_count(C.byref(self.s), C.byref(n), C.byref(p)), "count")
        return n.value, p.value

    def enumerate(self):
        n, _ = self.count()
        out = {k: np.zeros(n, np.int32) for k in ("job", "type", "G", "S", "nplans")}
        self._check(self.L.oracle_enumerate(C.byref(self.s), *[_ptr(out[k]) for k in
                                                                ("job", "type", "G", "S", "nplans")]),
                    "enumerate")
        return out

    def split(self, j, t, S):
        b = np.zeros(S + 1, np.int32)
        self._check(self.L.oracle_split(C.byref(self.s), j, t, S, _ptr(b)), "split")
        return b

    def plan_cost(self, j, t, G, S, p):
        T = np.zeros(S, np.int64)
        sy = np.zeros(S, np.int64)
        mem = np.zeros(S, np.int64)
        ti = C.c_int64()
        fe = C.c_int32()
        self._check(self.L.oracle_plan_cost(C.byref(self.s), j, t, G, S, p, _ptr(T), _ptr(sy),
                                            _ptr(mem), C.byref(ti), C.byref(fe)), "plan_cost")
        return dict(T=T, sync=sy, mem=mem, t_iter=ti.value, feasible=bool(fe.value))

    def estimate(self, cells, c0=0, c1=None):
        n = len(cells["job"])
        c1 = n if c1 is None else c1
        t_ns = np.zeros(c1 - c0, np.int64)
        plan = np.zeros(c1 - c0, np.int32)
        self._check(self.L.oracle_estimate(C.byref(self.s), *[_ptr(cells[k]) for k in
                                                              ("job", "type", "G", "S", "nplans")],
                                           C.c_int64(c0), C.c_int64(c1), _ptr(t_ns), _ptr(plan)),
                    "estimate")
        return t_ns, plan

    def estimate_assembled(self, cells, mode, form, c0=0, c1=None, kstride=None):
        n = len(cells["job"])
        c1 = n if c1 is None else c1
        kstride = int(cells["S"].max()) if kstride is None else kstride
        t_ns = np.zeros(c1 - c0, np.int64)
        bidx = np.zeros(c1 - c0, np.int32)
        sk = np.zeros((c1 - c0) * kstride, np.int8)
        self._check(self.L.oracle_estimate_assembled(
            C.byref(self.s), mode, form, *[_ptr(cells[k]) for k in ("job", "type", "G", "S")],
            C.c_int64(c0), C.c_int64(c1), _ptr(t_ns), _ptr(bidx), _ptr(sk), kstride),
            "estimate_assembled")
        return t_ns, bidx, sk.reshape(c1 - c0, kstride)

    def assembled_cost(self, form, j, t, G, S, bi, stage_k):
        ks = np.ascontiguousarray(stage_k[:S], np.int8)
        lat, fe = C.c_int64(), C.c_int32()
        self._check(self.L.oracle_assembled_cost(C.byref(self.s), form, j, t, G, S, bi, _ptr(ks),
                                                 C.byref(lat), C.byref(fe)), "assembled_cost")
        return lat.value, bool(fe.value)

    def tune_assembled(self, cells, form, favor, c0=0, c1=None):
        n = len(cells["job"])
        c1 = n if c1 is None else c1
        favor = np.ascontiguousarray(favor, np.int8)
        kstride = favor.shape[1]
        t_ns = np.zeros(c1 - c0, np.int64)
        bidx = np.zeros(c1 - c0, np.int32)
        sk = np.zeros((c1 - c0) * kstride, np.int8)
        self._check(self.L.oracle_tune_assembled(
            C.byref(self.s), form, *[_ptr(cells[k]) for k in ("job", "type", "G", "S")],
            C.c_int64(c0), C.c_int64(c1), _ptr(favor), kstride, _ptr(t_ns), _ptr(bidx), _ptr(sk)),
            "tune_assembled")
        return t_ns, bidx, sk.reshape(c1 - c0, kstride)

    def paper_stages(self, j, t, G, S):
        """NEXT-2: (cuts bounds[S+1], GPUs per stage g[S]) of Cell (j, t, G, S)."""
        b = np.zeros(S + 1, np.int32)
        g = np.zeros(S, np.int32)
        self._check(self.L.oracle_paper_stages(C.byref(self.s), j, t, G, S, _ptr(b), _ptr(g)),
                    "paper_stages")
        return b, g

    def paper_fractional(self, j, t, G, S, bounds):
        """NEXT-2: fractional GPUs G F_s / F of the stages of `bounds` as (num[S], den)."""
        b = np.ascontiguousarray(bounds, np.int32)
        num = np.zeros(S, np.int64)
        den = C.c_int64()
        self._check(self.L.oracle_paper_fractional(C.byref(self.s), j, t, G, S, _ptr(b), _ptr(num),
                                                   C.byref(den)), "paper_fractional")
        return num, den.value

    def paper_plan_cost(self, j, t, S, bounds, g, p):
        b = np.ascontiguousarray(bounds, np.int32)
        gg = np.ascontiguousarray(g, np.int32)
        ti, fe = C.c_int64(), C.c_int32()
        self._check(self.L.oracle_paper_plan_cost(C.byref(self.s), j, t, S, _ptr(b), _ptr(gg), p,
                                                  C.byref(ti), C.byref(fe)), "paper_plan_cost")
        return ti.value, bool(fe.value)

    def estimate_paper(self, cells, c0=0, c1=None, kstride=None):
        n = len(cells["job"])
        c1 = n if c1 is None else c1
        kstride = int(cells["S"].max()) if kstride is None else kstride
        t_ns = np.zeros(c1 - c0, np.int64)
        plan = np.zeros(c1 - c0, np.int32)
        lg = np.zeros((c1 - c0) * kstride, np.int8)
        self._check(self.L.oracle_estimate_paper(
            C.byref(self.s), *[_ptr(cells[k]) for k in ("job", "type", "G", "S")],
            C.c_int64(c0), C.c_int64(c1), _ptr(t_ns), _ptr(plan), _ptr(lg), kstride),
            "estimate_paper")
        return t_ns, plan, lg.reshape(c1 - c0, kstride)

    def round_state(self, cells, t_ns, free_in, run_cell=None, active=None, policy=0,
                    t_max=None):
        """NEXT-4 round from a state; policy bit 0 = NA, bit 1 = NH (ablations, R-11);
        t_max: per-job deadline bound on an option's T (R-12), None = no deadlines."""
        J, T = self.pr.n_jobs, self.pr.n_types
        dec = np.zeros(J, np.int64)
        fa = np.zeros(T, np.int32)
        tot = C.c_double()
        fi = np.ascontiguousarray(free_in, np.int32)
        rc, rcp = _opt_ptr(run_cell, np.int64)
        ac, acp = _opt_ptr(active, np.uint8)
        tm, tmp = _opt_ptr(t_max, np.int64)
        t_ns = np.ascontiguousarray(t_ns, np.int64)
        self._check(self.L.oracle_round_policy(
            C.byref(self.s), C.c_int64(len(t_ns)), *[_ptr(cells[k]) for k in ("job", "type", "G", "S")],
            _ptr(t_ns), _ptr(fi), rcp, acp, C.c_int32(policy), tmp, _ptr(dec), _ptr(fa),
            C.byref(tot)),
            "round_state")
        return dec, fa, tot.value

    def round(self, cells, t_ns, free_in=None):
        J, T = self.pr.n_jobs, self.pr.n_types
        dec = np.zeros(J, np.int64)
        fa = np.zeros(T, np.int32)
        tot = C.c_double()
        fi = None if free_in is None else np.ascontiguousarray(free_in, np.int32)
        t_ns = np.ascontiguousarray(t_ns, np.int64)
        self._check(self.L.oracle_round(C.byref(self.s), C.c_int64(len(t_ns)),
                                        *[_ptr(cells[k]) for k in ("job", "type", "G", "S")],
                                        _ptr(t_ns), None if fi is None else _ptr(fi), _ptr(dec),
                                        _ptr(fa), C.byref(tot)), "round")
        return dec, fa, tot.value


def _opt_ptr(a, dtype):
    if a is None:
        return None, None
    a = np.ascontiguousarray(a, dtype)
    return a, _ptr(a)


def tune_choices(g, tp_favour):
    ks = np.zeros(16, np.int32)
    n = lib().oracle_tune_choices(g, int(tp_favour), _ptr(ks))
    return [int(k) for k in ks[:n]]


def paper_round_pow2(num, den):
    """NEXT-2: num/den rounded to the nearest power of two (ties up, >= 1)."""
    f = lib().oracle_paper_round_pow2
    f.restype = C.c_int32
    f.argtypes = [C.c_int64, C.c_int64]
    return int(f(num, den))


def comm(kind, p, alpha, beta, V, n=1):
    return lib().oracle_comm(kind, p, alpha, beta, V, n)
