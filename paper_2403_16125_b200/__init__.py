"""paper_2403_16125_b200 -- B200-native Crius Cell estimator (arXiv 2403.16125).

Thin Python binding of libcrius (include/crius.h): argument marshalling only.
Every step of the hot path -- Cell enumeration, stage DP, plan cost, per-Cell
argmin, scheduling round, result compaction -- runs in the library's CUDA
kernels.  PyTorch provides device memory, streams and process groups.  There
is no CPU fallback: if libcrius.so is missing or no GPU is present, calls raise.

    from paper_2403_16125_b200 import Crius, workload
    pr = workload.make_config(4)
    with Crius(pr) as cr:
        n_cells, n_plans, _ = cr.enumerate()
        res = cr.estimate()                      # [n_cells, 2] int64 records on the GPU
        dec, free_after, total = cr.schedule_round(res)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import workload  # noqa: F401  (seeded inputs; none of the method's arithmetic)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CRIUS_LIB") or os.path.join(HERE, "libcrius.so")
INF = np.iinfo(np.int64).max
RECORD_BYTES = 16

STATUS = {0: "OK", 2: "EINVAL", 3: "EINFEASIBLE", 4: "ECUDA", 5: "ENOMEM", 6: "ESTATE"}


class CriusError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"crius {STATUS.get(code, code)}: {msg}")
        self.code = code


class _Cluster(C.Structure):
    _fields_ = [("n_types", C.c_int32), ("capacity", C.c_void_p), ("gpus_per_node", C.c_void_p),
                ("mem_bytes", C.c_void_p), ("alpha_intra_ns", C.c_void_p),
                ("beta_intra_ns_per_mib", C.c_void_p), ("alpha_inter_ns", C.c_void_p),
                ("beta_inter_ns_per_mib", C.c_void_p)]


class _Jobs(C.Structure):
    _fields_ = [("n_jobs", C.c_int32), ("k_max", C.c_int32), ("job_id", C.c_void_p),
                ("submit_time", C.c_void_p), ("n_gpus_req", C.c_void_p),
                ("global_batch", C.c_void_p), ("k_state", C.c_void_p), ("n_layers", C.c_void_p),
                ("layer_off", C.c_void_p), ("compute_ns", C.c_void_p), ("param_bytes", C.c_void_p),
                ("act_bytes", C.c_void_p), ("boundary_bytes", C.c_void_p), ("tp_bytes", C.c_void_p),
                ("tp_calls", C.c_void_p)]


class _Config(C.Structure):
    _fields_ = [("gpu_set", C.c_int32), ("s_max", C.c_int32), ("g_max", C.c_int32),
                ("b_mode", C.c_int32), ("b_count", C.c_int32), ("b_values", C.c_void_p),
                ("search_depth", C.c_int32)]


class _Assembly(C.Structure):
    _fields_ = [("mode", C.c_int32), ("pipeline_form", C.c_int32)]


class _CellView(C.Structure):
    _fields_ = [("n_cells", C.c_int64), ("n_cell_plans", C.c_int64), ("n_units", C.c_int64),
                ("job", C.c_void_p), ("type", C.c_void_p), ("G", C.c_void_p), ("S", C.c_void_p),
                ("nplans", C.c_void_p), ("plan_off", C.c_void_p), ("unit_cell_begin", C.c_void_p),
                ("unit_plan_begin", C.c_void_p)]


EXPORTS = ["crius_load_profiles", "crius_update_profiles", "crius_update_profiles_range",
           "crius_enumerate_cells", "crius_cells",
           "crius_split_stride", "crius_max_stages", "crius_partition_units",
           "crius_estimate_cells", "crius_update_estimate", "crius_estimate_assembled", "crius_tune_assembled",
           "crius_estimate_paper_stages",
           "crius_compact_gathered", "crius_exchange_init", "crius_exchange_open",
           "crius_estimate_exchange", "crius_exchange_wait", "crius_exchange_close",
           "crius_schedule_round", "crius_schedule_round_state",
           "crius_round_stats", "crius_set_round_policy", "crius_set_deadline_bounds",
           "crius_kernel_launches",
           "crius_last_error", "crius_destroy"]

_lib = None


def lib():
    """Load libcrius.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2403_16125_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.crius_load_profiles.argtypes = [C.POINTER(vp), C.POINTER(_Cluster), C.POINTER(_Jobs),
                                          C.POINTER(_Config), i32, vp]
        L.crius_update_profiles.argtypes = [vp, C.POINTER(_Cluster), C.POINTER(_Jobs), vp]
        L.crius_update_profiles_range.argtypes = [vp, C.POINTER(_Cluster), C.POINTER(_Jobs), i32,
                                                  i32, vp]
        L.crius_enumerate_cells.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), vp]
        L.crius_cells.argtypes = [vp, C.POINTER(_CellView)]
        L.crius_split_stride.argtypes = [vp]
        L.crius_split_stride.restype = i32
        L.crius_partition_units.argtypes = [vp, i32, vp, vp, vp]
        L.crius_estimate_cells.argtypes = [vp, i64, i64, vp, vp, vp]
        if hasattr(L, "crius_update_estimate"):  # (absent from older builds used in A/B runs)
            L.crius_update_estimate.argtypes = [vp, C.POINTER(_Cluster), C.POINTER(_Jobs), i32, vp,
                                                i64, vp, C.POINTER(i64), C.POINTER(i64),
                                                C.POINTER(i64), vp]
        L.crius_estimate_assembled.argtypes = [vp, C.POINTER(_Assembly), i64, i64, vp, vp, vp]
        L.crius_tune_assembled.argtypes = [vp, i32, i64, i64, vp, vp, vp, vp]
        L.crius_estimate_paper_stages.argtypes = [vp, i64, i64, vp, vp, vp, vp]
        L.crius_max_stages.argtypes = [vp]
        L.crius_max_stages.restype = i32
        L.crius_compact_gathered.argtypes = [vp, vp, i64, i32, vp, vp, vp]
        L.crius_exchange_init.argtypes = [vp, i32, i32, i64, vp]
        L.crius_exchange_open.argtypes = [vp, vp]
        L.crius_estimate_exchange.argtypes = [vp, i64, i64, vp]
        L.crius_exchange_wait.argtypes = [vp, C.POINTER(vp), vp]
        L.crius_exchange_close.argtypes = [vp]
        L.crius_schedule_round.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.crius_schedule_round_state.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.crius_round_stats.argtypes = [vp, vp, vp]
        L.crius_set_round_policy.argtypes = [vp, i32]
        L.crius_set_deadline_bounds.argtypes = [vp, vp, vp]
        L.crius_kernel_launches.argtypes = [vp]
        L.crius_kernel_launches.restype = i64
        L.crius_last_error.restype = C.c_char_p
        L.crius_destroy.argtypes = [vp]
        L.crius_destroy.restype = None
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise CriusError(code, lib().crius_last_error().decode())


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


class _DevArray:
    """Zero-copy __cuda_array_interface__ wrapper of a library-owned device array."""

    def __init__(self, ptr, n, typestr, device):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3}
        self.device = device


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Crius:
    """One libcrius context on one GPU (PAPER.md:204-217 estimator + scheduler)."""

    def __init__(self, pr, device=None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise CriusError(4, "no CUDA device (there is no CPU fallback)")
        self.torch = torch
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.pr = pr
        self._keep = []
        cl, jb, cf = self._structs(pr)
        ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib().crius_load_profiles(C.byref(ctx), C.byref(cl), C.byref(jb), C.byref(cf),
                                             self.device, _stream_handle(stream)))
        self.ctx = ctx
        self.n_cells = self.n_plans = self.n_units = None

    # -- marshalling --------------------------------------------------------
    def _arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        self._keep.append(a)
        return _ptr(a)

    def _structs(self, pr):
        self._keep = []
        cl = _Cluster(pr.n_types, self._arr(pr.cap, np.int32), self._arr(pr.gpn, np.int32),
                      self._arr(pr.mem, np.int64), self._arr(pr.alpha_in, np.int64),
                      self._arr(pr.beta_in, np.int64), self._arr(pr.alpha_x, np.int64),
                      self._arr(pr.beta_x, np.int64))
        jb = _Jobs(pr.n_jobs, pr.k_max, self._arr(pr.job_id, np.int64),
                   self._arr(pr.submit, np.int64), self._arr(pr.ng, np.int32),
                   self._arr(pr.gb, np.int32), self._arr(pr.kst, np.int32),
                   self._arr(pr.n_layers, np.int32), self._arr(pr.layer_off, np.int64),
                   self._arr(pr.c, np.int32), self._arr(pr.w, np.int64),
                   self._arr(pr.act, np.int64), self._arr(pr.bnd, np.int64),
                   self._arr(pr.tpv, np.int64), self._arr(pr.tpn, np.int32))
        bv = np.ascontiguousarray(pr.b_values if pr.b_mode == 1 else np.zeros(1), np.int32)
        cf = _Config(pr.gpu_set, pr.s_max, pr.g_max, pr.b_mode,
                     int(pr.b_values.size) if pr.b_mode == 1 else 0, self._arr(bv, np.int32),
                     pr.depth)
        return cl, jb, cf

    # -- the C-ABI calls ------------------------------------------------------
    def update(self, pr, job_begin=None, job_end=None, stream=None):
        """New profile values (same shapes); per-layer rows only for jobs
        [job_begin, job_end) when a range is given (a rank's shard)."""
        cl, jb, _ = self._structs(pr)
        if job_begin is None:
            _check(lib().crius_update_profiles(self.ctx, C.byref(cl), C.byref(jb),
                                               _stream_handle(stream)))
        else:
            _check(lib().crius_update_profiles_range(self.ctx, C.byref(cl), C.byref(jb),
                                                     int(job_begin), int(job_end),
                                                     _stream_handle(stream)))
        self.pr = pr

    def enumerate(self, stream=None):
        n, p, u = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().crius_enumerate_cells(self.ctx, C.byref(n), C.byref(p), C.byref(u),
                                           _stream_handle(stream)))
        self.n_cells, self.n_plans, self.n_units = n.value, p.value, u.value
        return self.n_cells, self.n_plans, self.n_units

    def cells(self):
        """Device Cell table as zero-copy torch tensors."""
        v = _CellView()
        _check(lib().crius_cells(self.ctx, C.byref(v)))
        t = self.torch
        dev = f"cuda:{self.device}"

        def wrap(ptr, n, ts):
            return t.as_tensor(_DevArray(ptr, n, ts, dev), device=dev)

        n, u = v.n_cells, v.n_units
        return dict(job=wrap(v.job, n, "<i4"), type=wrap(v.type, n, "<i4"), G=wrap(v.G, n, "<i4"),
                    S=wrap(v.S, n, "<i4"), nplans=wrap(v.nplans, n, "<i4"),
                    plan_off=wrap(v.plan_off, n, "<i8"),
                    unit_cell_begin=wrap(v.unit_cell_begin, u + 1, "<i8"),
                    unit_plan_begin=wrap(v.unit_plan_begin, u + 1, "<i8"))

    def split_stride(self):
        return lib().crius_split_stride(self.ctx)

    def partition(self, world, stream=None):
        ub = np.zeros(world + 1, np.int64)
        cb = np.zeros(world + 1, np.int64)
        _check(lib().crius_partition_units(self.ctx, world, _ptr(ub), _ptr(cb),
                                           _stream_handle(stream)))
        return ub, cb

    def new_results(self, n):
        return self.torch.empty((max(int(n), 1), 2), dtype=self.torch.int64,
                                device=f"cuda:{self.device}")

    def estimate(self, unit_begin=0, unit_end=None, out=None, splits=None, stream=None):
        """Records of Cells [ucb[unit_begin], ucb[unit_end]) into `out` ([n, 2] int64 on the GPU)."""
        if self.n_cells is None:
            self.enumerate(stream)
        unit_end = self.n_units if unit_end is None else unit_end
        if out is None:
            out = self.new_results(self.n_cells)
        sp = C.c_void_p(splits.data_ptr()) if splits is not None else None
        _check(lib().crius_estimate_cells(self.ctx, int(unit_begin), int(unit_end),
                                          C.c_void_p(out.data_ptr()), sp, _stream_handle(stream)))
        return out

    def update_estimate(self, pr, chunks=4, out=None, splits=None, stream=None):
        """New profile values from host memory -> every Cell's record, with the
        per-layer row upload pipelined against the estimate in `chunks` job
        ranges (crius_update_estimate; pinned host arrays overlap).  Returns the
        [n_cells, 2] records (global Cell order)."""
        cl, jb, _ = self._structs(pr)
        if out is None:
            if self.n_cells is None:
                self.enumerate(stream)
            out = self.new_results(self.n_cells)
        n, p, u = C.c_int64(), C.c_int64(), C.c_int64()
        sp = C.c_void_p(splits.data_ptr()) if splits is not None else None
        st = lib().crius_update_estimate(self.ctx, C.byref(cl), C.byref(jb), int(chunks),
                                         C.c_void_p(out.data_ptr()), int(out.shape[0]), sp,
                                         C.byref(n), C.byref(p), C.byref(u), _stream_handle(stream))
        if st == 2 and n.value > out.shape[0]:  # more Cells than `out` holds: grow, call again
            out = self.new_results(n.value)
            st = lib().crius_update_estimate(self.ctx, C.byref(cl), C.byref(jb), int(chunks),
                                             C.c_void_p(out.data_ptr()), int(out.shape[0]), sp,
                                             C.byref(n), C.byref(p), C.byref(u),
                                             _stream_handle(stream))
        _check(st)
        self.pr = pr
        self.n_cells, self.n_plans, self.n_units = n.value, p.value, u.value
        return out

    def max_stages(self):
        return lib().crius_max_stages(self.ctx)

    def estimate_assembled(self, mode=1, form=1, unit_begin=0, unit_end=None, out=None,
                           stage_tp=None, stream=None):
        """NEXT-1 per-stage assembly (mode 1: DP-only/TP-only per stage, the
        paper's 2^S plans; mode 2: every factorisation per stage; form 1: the
        paper's (B-1)(T_s* - T_comm) steady state).  Records as estimate();
        stage_tp: optional int8 [n_cells, max_stages] device tensor."""
        if self.n_cells is None:
            self.enumerate(stream)
        unit_end = self.n_units if unit_end is None else unit_end
        if out is None:
            out = self.new_results(self.n_cells)
        cfg = _Assembly(mode, form)
        sp = C.c_void_p(stage_tp.data_ptr()) if stage_tp is not None else None
        _check(lib().crius_estimate_assembled(self.ctx, C.byref(cfg), int(unit_begin),
                                              int(unit_end), C.c_void_p(out.data_ptr()), sp,
                                              _stream_handle(stream)))
        return out

    def estimate_paper_stages(self, unit_begin=0, unit_end=None, out=None, splits=None,
                              stage_lg=None, stream=None):
        """NEXT-2: the paper's stage determination (cuts at the smallest boundary
        bytes, FLOP-proportional power-of-two GPUs per stage) and the best plan
        (uniform tp, per-stage dp).  Records as estimate(); splits as estimate();
        stage_lg: optional int8 [n_cells, max_stages] device tensor (log2 g_s)."""
        if self.n_cells is None:
            self.enumerate(stream)
        unit_end = self.n_units if unit_end is None else unit_end
        if out is None:
            out = self.new_results(self.n_cells)
        sp = C.c_void_p(splits.data_ptr()) if splits is not None else None
        lg = C.c_void_p(stage_lg.data_ptr()) if stage_lg is not None else None
        _check(lib().crius_estimate_paper_stages(self.ctx, int(unit_begin), int(unit_end),
                                                 C.c_void_p(out.data_ptr()), sp, lg,
                                                 _stream_handle(stream)))
        return out

    def tune_assembled(self, favor, form=1, unit_begin=0, unit_end=None, out=None, stage_tp=None,
                       stream=None):
        """NEXT-3 Cell-guided tuning: favor = int8 [n_cells, max_stages] device tensor
        (log2 tp per stage of the estimated plan, e.g. estimate_assembled's stage_tp)."""
        if self.n_cells is None:
            self.enumerate(stream)
        unit_end = self.n_units if unit_end is None else unit_end
        if out is None:
            out = self.new_results(self.n_cells)
        sp = C.c_void_p(stage_tp.data_ptr()) if stage_tp is not None else None
        _check(lib().crius_tune_assembled(self.ctx, form, int(unit_begin), int(unit_end),
                                          C.c_void_p(favor.data_ptr()), C.c_void_p(out.data_ptr()),
                                          sp, _stream_handle(stream)))
        return out

    def compact(self, gathered, chunk_stride, world, cell_begin, out=None, stream=None):
        if out is None:
            out = self.new_results(self.n_cells)
        cb = np.ascontiguousarray(cell_begin, np.int64)
        _check(lib().crius_compact_gathered(self.ctx, C.c_void_p(gathered.data_ptr()),
                                            int(chunk_stride), int(world), _ptr(cb),
                                            C.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    # ---- fused exchange over NVLink peer memory (crius_exchange_*)
    def exchange_init(self, rank, world, capacity=None):
        """Allocate this rank's exchange window; returns its 64-byte IPC handle."""
        cap = int(capacity if capacity is not None else max(self.n_cells or 1, 1))
        h = (C.c_uint8 * 64)()
        _check(lib().crius_exchange_init(self.ctx, int(rank), int(world), cap, h))
        return bytes(h)

    def exchange_open(self, handles):
        """handles: every rank's 64-byte handle concatenated in rank order."""
        buf = (C.c_uint8 * len(handles)).from_buffer_copy(bytes(handles))
        _check(lib().crius_exchange_open(self.ctx, buf))

    def estimate_exchange(self, unit_begin, unit_end, stream=None):
        """Estimate [unit_begin, unit_end) and store every record into every rank's window."""
        _check(lib().crius_estimate_exchange(self.ctx, int(unit_begin), int(unit_end),
                                             _stream_handle(stream)))

    def exchange_wait(self, stream=None):
        """Enqueue the wait for every rank's records; returns the window half of
        this step as an [n_cells, 2] int64 device tensor (a view, no copy)."""
        p = C.c_void_p()
        _check(lib().crius_exchange_wait(self.ctx, C.byref(p), _stream_handle(stream)))
        return self.torch.as_tensor(_DevView(p.value, int(self.n_cells)),
                                    device=f"cuda:{self.device}")

    def exchange_close(self):
        _check(lib().crius_exchange_close(self.ctx))

    def schedule_round(self, results, free=None, stream=None):
        J, T = self.pr.n_jobs, self.pr.n_types
        dec = np.zeros(J, np.int64)
        fa = np.zeros(T, np.int32)
        tot = C.c_double()
        fr = None if free is None else self._arr(free, np.int32)
        _check(lib().crius_schedule_round(self.ctx, C.c_void_p(results.data_ptr()), fr, _ptr(dec),
                                          _ptr(fa), C.byref(tot), _stream_handle(stream)))
        return dec, fa, tot.value

    def schedule_round_state(self, results, free, run_cell=None, active=None, stream=None):
        """NEXT-4: one round from a cluster state (running jobs keep/may move their
        Cells; inactive jobs are skipped with decision -3)."""
        J, T = self.pr.n_jobs, self.pr.n_types
        dec = np.zeros(J, np.int64)
        fa = np.zeros(T, np.int32)
        tot = C.c_double()
        fr = np.ascontiguousarray(free, np.int32)
        rc = None if run_cell is None else np.ascontiguousarray(run_cell, np.int64)
        ac = None if active is None else np.ascontiguousarray(active, np.uint8)
        _check(lib().crius_schedule_round_state(
            self.ctx, C.c_void_p(results.data_ptr()), _ptr(fr), None if rc is None else _ptr(rc),
            None if ac is None else _ptr(ac), _ptr(dec), _ptr(fa), C.byref(tot),
            _stream_handle(stream)))
        return dec, fa, tot.value

    def set_round_policy(self, policy):
        """NEXT-4 ablations: 0 full round, 1 NA (no GPU-count change), 2 NH (no
        GPU-type change of admitted jobs), 3 both."""
        _check(lib().crius_set_round_policy(self.ctx, int(policy)))

    def set_deadline_bounds(self, t_max, stream=None):
        """Per-job bound on an option's iteration time (ns) for later rounds
        (deadline-aware scheduling, R-12); None removes it."""
        if t_max is None:
            _check(lib().crius_set_deadline_bounds(self.ctx, None, _stream_handle(stream)))
            return
        a = np.ascontiguousarray(t_max, np.int64)
        if a.shape != (self.pr.n_jobs,):
            raise ValueError("t_max must have one entry per job")
        _check(lib().crius_set_deadline_bounds(self.ctx, _ptr(a), _stream_handle(stream)))
        # the upload is asynchronous: keep the host array alive until it has run
        self.torch.cuda.synchronize(self.device)

    def round_stats(self, stream=None):
        out = np.zeros(32, np.int64)
        _check(lib().crius_round_stats(self.ctx, _ptr(out), _stream_handle(stream)))
        keys = {0: "phaseA_batches", 1: "seq_recomputes", 2: "seq_cycles", 3: "phaseA_cycles",
                4: "phaseB_cycles", 5: "admitted", 6: "scale_admits", 7: "phaseB_batches",
                8: "batch_direct_cycles", 9: "batch_scale_cycles", 10: "batch_commit_cycles",
                11: "stale_caches", 12: "other_type_evals", 13: "seq_invalidations",
                14: "records_in_smem", 15: "records_bound", 16: "seq_prep_cycles",
                17: "seq_move_cycles", 18: "seq_tail_cycles", 19: "seq_rescans", 20: "seq_entries",
                21: "top_refills", 22: "seq_type_runs", 23: "seq_top_refresh_cycles",
                25: "seq_stale_types",
                28: "cta_barriers"}
        return {k: int(out[i]) for i, k in keys.items()}

    def launches(self):
        return lib().crius_kernel_launches(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            lib().crius_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DevView:
    """[n, 2] int64 view of library-owned device memory (CUDA array interface)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (max(n, 1), 2), "typestr": "<i8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}


def decode(results):
    """[n, 2] int64 device records -> (t_ns int64, plan int32, flags int32) numpy."""
    r = results.cpu().numpy()
    t_ns = r[:, 0].copy()
    pf = np.ascontiguousarray(r[:, 1]).view(np.int32).reshape(-1, 2)
    return t_ns, pf[:, 0].copy(), pf[:, 1].copy()
