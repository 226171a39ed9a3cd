"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of the `orc_*` ABI (oracle/edx_oracle.h).  The same class loads
either the plain-C restatement (oracle/liboracle.so, kind="port") or the
compiled, unmodified reference (oracle/_ref/libedx_ref.so, kind="reference").
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libedx_ref.so")

ORC_OK, ORC_INVALID_ARGUMENT, ORC_LOGIC_ERROR, ORC_RUNTIME_ERROR = 0, 1, 2, 3


class OracleInvalidArgument(ValueError):
    pass


class OracleLogicError(RuntimeError):
    pass


class OracleRuntimeError(RuntimeError):
    pass


_EXC = {ORC_INVALID_ARGUMENT: OracleInvalidArgument, ORC_LOGIC_ERROR: OracleLogicError,
        ORC_RUNTIME_ERROR: OracleRuntimeError}


class ClusterConfigC(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("bandwidths_bps", C.POINTER(C.c_double)),
                ("n_bandwidths", C.c_int32), ("reserved", C.c_int32),
                ("d_tran_bytes", C.c_uint64), ("cache_capacity", C.c_uint64),
                ("alpha", C.c_double)]


class ReportC(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("miss_pull", C.c_uint64),
                ("update_push", C.c_uint64), ("evict_push", C.c_uint64),
                ("hits", C.c_uint64), ("lookups", C.c_uint64), ("cost_s", C.c_double),
                ("miss_pull_w", C.POINTER(C.c_uint64)), ("update_push_w", C.POINTER(C.c_uint64)),
                ("evict_push_w", C.POINTER(C.c_uint64)), ("cost_w", C.POINTER(C.c_double))]


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all" if ref else "liboracle.so"], check=True)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


class Cfg:
    """Mirror of embdispatch::ClusterConfig (types.hpp:71-82)."""

    def __init__(self, n, m, bw, d_tran=2048, cap=64, alpha=1.0):
        self.n, self.m, self.alpha = int(n), int(m), float(alpha)
        self.bw = np.ascontiguousarray(np.asarray(bw, dtype=np.float64))
        self.d_tran, self.cap = int(d_tran), int(cap)

    def c(self):
        return ClusterConfigC(self.n, self.m, self.bw.ctypes.data_as(C.POINTER(C.c_double)),
                              len(self.bw), 0, self.d_tran, self.cap, self.alpha)


class Report:
    def __init__(self, n):
        self.miss_pull_w = np.zeros(n, np.uint64)
        self.update_push_w = np.zeros(n, np.uint64)
        self.evict_push_w = np.zeros(n, np.uint64)
        self.cost_w = np.zeros(n, np.float64)
        self.c = ReportC(0, 0, 0, 0, 0, 0, 0.0, _p(self.miss_pull_w, C.c_uint64),
                         _p(self.update_push_w, C.c_uint64), _p(self.evict_push_w, C.c_uint64),
                         _p(self.cost_w, C.c_double))

    def as_dict(self):
        c = self.c
        return dict(iteration=c.iteration, miss_pull=c.miss_pull, update_push=c.update_push,
                    evict_push=c.evict_push, hits=c.hits, lookups=c.lookups, cost_s=c.cost_s,
                    miss_pull_w=self.miss_pull_w.tolist(),
                    update_push_w=self.update_push_w.tolist(),
                    evict_push_w=self.evict_push_w.tolist(), cost_w=self.cost_w.tolist())


class Oracle:
    def __init__(self, kind: str = "port"):
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.kind = kind
        self.lib = L = C.CDLL(path)
        vp, u64, i32, dbl = C.c_void_p, C.c_uint64, C.c_int32, C.c_double
        P = C.POINTER
        L.orc_last_error.restype = C.c_char_p
        L.orc_zipf_create.argtypes = [u64, u64, dbl, u64, u64, u64, P(vp)]
        L.orc_zipf_next.argtypes = [vp, P(C.c_uint32)]
        L.orc_zipf_destroy.argtypes = [vp]
        L.orc_zipf_reset.argtypes = [vp]
        L.orc_bench_matrix.argtypes = [u64, P(dbl)]
        L.orc_validate_config.argtypes = [P(ClusterConfigC), u64]
        L.orc_unit_costs.argtypes = [P(ClusterConfigC), P(dbl)]
        L.orc_build_matrix_snapshot.argtypes = [P(ClusterConfigC), P(C.c_uint32), P(u64), P(u64),
                                                P(u64), u64, P(C.c_uint32), P(u64), u64, P(dbl)]
        L.orc_expected_costs_sized.argtypes = [P(ClusterConfigC), P(C.c_uint32), P(u64), P(u64),
                                               u64, P(C.c_uint32), P(u64), u64, P(u64), P(dbl)]
        L.orc_hitgreedy_snapshot.argtypes = [P(ClusterConfigC), P(C.c_uint32), P(u64), P(u64), u64,
                                             P(C.c_uint32), P(u64), u64, P(i32)]
        L.orc_sim_hitgreedy.argtypes = [vp, P(C.c_uint32), P(u64), u64, P(i32)]
        L.orc_row_gap_key.argtypes = [u64, u64, P(dbl), u64, P(dbl)]
        L.orc_rows_by_gap.argtypes = [u64, u64, P(dbl), P(u64)]
        L.orc_hungarian.argtypes = [u64, P(dbl), P(u64), P(dbl)]
        L.orc_greedy_dispatch.argtypes = [u64, u64, P(dbl), P(u64), u64, P(i32), P(u64), P(i32)]
        L.orc_ecomix.argtypes = [P(ClusterConfigC), u64, u64, P(dbl), P(u64), P(i32)]
        L.orc_decision_cost.argtypes = [u64, u64, P(dbl), P(i32), P(dbl)]
        L.orc_sim_create.argtypes = [P(ClusterConfigC), P(vp)]
        L.orc_sim_destroy.argtypes = [vp]
        L.orc_sim_build_matrix.argtypes = [vp, P(C.c_uint32), P(u64), u64, P(dbl)]
        L.orc_sim_step.argtypes = [vp, P(C.c_uint32), P(u64), u64, P(i32), P(ReportC)]
        L.orc_sim_seed_entry.argtypes = [vp, C.c_uint32, i32, C.c_int, C.c_int]
        L.orc_sim_validate_consistency.argtypes = [vp]
        L.orc_sim_clock.argtypes = [vp]
        L.orc_sim_clock.restype = u64
        L.orc_sim_global_count.argtypes = [vp]
        L.orc_sim_global_count.restype = u64
        L.orc_sim_export_global.argtypes = [vp, P(C.c_uint32), P(u64), P(u64), P(u64)]
        L.orc_sim_cache_size.argtypes = [vp, i32]
        L.orc_sim_cache_size.restype = u64
        L.orc_sim_export_cache.argtypes = [vp, i32, P(C.c_uint32), P(C.c_uint8), P(C.c_uint32),
                                           P(C.c_uint32), P(u64)]
        L.orc_sim_cache_marks.argtypes = [vp, i32, P(C.c_uint32), P(u64)]
        L.orc_sim_import_state.argtypes = [vp, u64, u64, P(C.c_uint32), P(u64), P(u64), P(u64),
                                           P(u64), P(C.c_uint32), P(C.c_uint8), P(C.c_uint32),
                                           P(C.c_uint32), P(u64), P(C.c_uint32), P(u64)]
        L.orc_ref_iteration.argtypes = [vp, P(C.c_uint32), P(u64), u64, C.c_int, P(i32), P(dbl),
                                        P(ReportC), P(dbl)]
        L.orc_last_hungarian_steps.restype = u64
        L.orc_cache_create.argtypes = [u64, C.c_int, P(vp)]
        L.orc_cache_destroy.argtypes = [vp]
        L.orc_cache_touch.argtypes = [vp, C.c_uint32, C.c_int, u64, dbl]
        L.orc_cache_set_version.argtypes = [vp, C.c_uint32, C.c_int]
        L.orc_cache_erase.argtypes = [vp, C.c_uint32]
        L.orc_cache_select_victim.argtypes = [vp, P(C.c_uint32)]
        L.orc_cache_evict_for.argtypes = [vp, u64, P(C.c_uint32), u64, P(C.c_uint32), P(u64)]
        L.orc_cache_info.argtypes = [vp, P(u64), P(C.c_uint32)]
        L.orc_cache_export.argtypes = [vp, P(C.c_uint32), P(C.c_uint8), P(C.c_uint32),
                                       P(C.c_uint32), P(u64)]

    def _check(self, rc):
        if rc != ORC_OK:
            raise _EXC.get(rc, OracleRuntimeError)(self.lib.orc_last_error().decode())

    # ---- workload
    def zipf_batches(self, total, sample_len, s, iterations, seed, per_iteration):
        h = C.c_void_p()
        self._check(self.lib.orc_zipf_create(total, sample_len, s, iterations, seed,
                                             per_iteration, C.byref(h)))
        try:
            while True:
                ids = np.empty(per_iteration * sample_len, np.uint32)
                if not self.lib.orc_zipf_next(h, _p(ids, C.c_uint32)):
                    return
                yield ids
        finally:
            self.lib.orc_zipf_destroy(h)

    def trace_dump(self, path, schema_path, n, m, capacity):
        """Compiled reference only: TraceStream(path, cfg, schema) dumped as
        text by oracle/_ref/trace_dump (its own process: the reference's
        iostreams and numpy's C++ runtime do not share one safely); returns
        (True, text) or (False, message)."""
        import subprocess
        exe = os.path.join(os.path.dirname(REF_SO), "trace_dump")
        r = subprocess.run([exe, path, schema_path or "-", str(n), str(m), str(capacity)],
                           capture_output=True, check=True)
        head, _, body = r.stdout.partition(b"\n")
        return head == b"OK", body.decode("latin-1")

    def bench_matrix(self, k):
        out = np.empty(k * k, np.float64)
        self.lib.orc_bench_matrix(k, _p(out, C.c_double))
        return out.reshape(k, k)

    # ---- matrix level
    def validate_config(self, cfg: Cfg, max_len):
        self._check(self.lib.orc_validate_config(C.byref(cfg.c()), max_len))

    def unit_costs(self, cfg: Cfg):
        out = np.empty(cfg.n, np.float64)
        self._check(self.lib.orc_unit_costs(C.byref(cfg.c()), _p(out, C.c_double)))
        return out

    def build_matrix_snapshot(self, cfg: Cfg, snap, ids, offsets):
        """snap: dict id -> (owners, latest, resident)."""
        keys = np.array(sorted(snap), np.uint32)
        ow = np.array([snap[int(k)][0] for k in keys], np.uint64)
        la = np.array([snap[int(k)][1] for k in keys], np.uint64)
        re = np.array([snap[int(k)][2] for k in keys], np.uint64)
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        out = np.empty(max(R, 0) * cfg.n, np.float64)
        self._check(self.lib.orc_build_matrix_snapshot(
            C.byref(cfg.c()), _p(keys, C.c_uint32), _p(ow, C.c_uint64), _p(la, C.c_uint64),
            _p(re, C.c_uint64), len(keys), _p(ids, C.c_uint32), _p(offsets, C.c_uint64), R,
            _p(out, C.c_double)))
        return out.reshape(R, cfg.n)

    def expected_costs_sized(self, cfg: Cfg, snap, ids, offsets, sizes):
        """Every expected_cost cell with a SizeLookupFn; sizes[t] per id position."""
        keys = np.array(sorted(snap), np.uint32)
        ow = np.array([snap[int(k)][0] for k in keys], np.uint64)
        la = np.array([snap[int(k)][1] for k in keys], np.uint64)
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        sizes = np.ascontiguousarray(sizes, np.uint64)
        R = len(offsets) - 1
        out = np.empty(max(R, 0) * cfg.n, np.float64)
        self._check(self.lib.orc_expected_costs_sized(
            C.byref(cfg.c()), _p(keys, C.c_uint32), _p(ow, C.c_uint64), _p(la, C.c_uint64),
            len(keys), _p(ids, C.c_uint32), _p(offsets, C.c_uint64), R, _p(sizes, C.c_uint64),
            _p(out, C.c_double)))
        return out.reshape(R, cfg.n)

    def hitgreedy_snapshot(self, cfg: Cfg, snap, ids, offsets):
        """baseline_hitgreedy (assign.hpp:346-392); snap: dict id -> (owners, latest, ...)."""
        keys = np.array(sorted(snap), np.uint32)
        ow = np.array([snap[int(k)][0] for k in keys], np.uint64)
        la = np.array([snap[int(k)][1] for k in keys], np.uint64)
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        dec = np.empty(max(R, 1), np.int32)
        self._check(self.lib.orc_hitgreedy_snapshot(
            C.byref(cfg.c()), _p(keys, C.c_uint32), _p(ow, C.c_uint64), _p(la, C.c_uint64),
            len(keys), _p(ids, C.c_uint32), _p(offsets, C.c_uint64), R, _p(dec, C.c_int32)))
        return dec[:R]

    def row_gap_key(self, mat, row):
        mat = np.ascontiguousarray(mat, np.float64)
        out = C.c_double()
        self._check(self.lib.orc_row_gap_key(mat.shape[0], mat.shape[1], _p(mat, C.c_double),
                                             row, C.byref(out)))
        return out.value

    def rows_by_gap(self, mat):
        mat = np.ascontiguousarray(mat, np.float64)
        out = np.empty(mat.shape[0], np.uint64)
        self._check(self.lib.orc_rows_by_gap(mat.shape[0], mat.shape[1], _p(mat, C.c_double),
                                             _p(out, C.c_uint64)))
        return out

    def hungarian(self, sq):
        sq = np.ascontiguousarray(sq, np.float64)
        k = sq.shape[0] if sq.ndim == 2 else int(round(len(sq) ** 0.5))
        cols = np.empty(k, np.uint64)
        total = C.c_double()
        self._check(self.lib.orc_hungarian(k, _p(sq, C.c_double), _p(cols, C.c_uint64),
                                           C.byref(total)))
        return cols, total.value

    def greedy_dispatch(self, mat, order, capacity):
        mat = np.ascontiguousarray(mat, np.float64)
        order = np.ascontiguousarray(order, np.uint64)
        cap = np.ascontiguousarray(capacity, np.int32)
        rows = np.empty(len(order), np.uint64)
        workers = np.empty(len(order), np.int32)
        self._check(self.lib.orc_greedy_dispatch(mat.shape[0], mat.shape[1], _p(mat, C.c_double),
                                                 _p(order, C.c_uint64), len(order),
                                                 _p(cap, C.c_int32), _p(rows, C.c_uint64),
                                                 _p(workers, C.c_int32)))
        return rows, workers

    def ecomix(self, cfg: Cfg, mat, row_ids=None):
        mat = np.ascontiguousarray(mat, np.float64)
        dec = np.empty(mat.shape[0], np.int32)
        rid = None if row_ids is None else np.ascontiguousarray(row_ids, np.uint64)
        self._check(self.lib.orc_ecomix(C.byref(cfg.c()), mat.shape[0], mat.shape[1],
                                        _p(mat, C.c_double), _p(rid, C.c_uint64),
                                        _p(dec, C.c_int32)))
        return dec

    def decision_cost(self, mat, dec):
        mat = np.ascontiguousarray(mat, np.float64)
        dec = np.ascontiguousarray(dec, np.int32)
        out = C.c_double()
        self._check(self.lib.orc_decision_cost(mat.shape[0], mat.shape[1], _p(mat, C.c_double),
                                               _p(dec, C.c_int32), C.byref(out)))
        return out.value

    def hungarian_steps(self):
        return int(self.lib.orc_last_hungarian_steps())

    def sim(self, cfg: Cfg):
        return Sim(self, cfg)

    def cache(self, capacity, policy=0):
        return Cache(self, capacity, policy)


def state_arrays(state, n):
    """canonical_state()-format state -> the flat arrays of orc_sim_import_state
    / edx_engine_import_state."""
    glob, caches = state
    glob = np.asarray(glob, np.uint64).reshape(-1, 4)
    assert len(caches) == n
    ents = [np.asarray(c[0], np.uint64).reshape(-1, 5) for c in caches]
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(e) for e in ents])
    cat = np.concatenate(ents) if ents else np.zeros((0, 5), np.uint64)
    c = np.ascontiguousarray
    return dict(g_ids=c(glob[:, 0].astype(np.uint32)), g_owners=c(glob[:, 1]),
                g_latest=c(glob[:, 2]), g_resident=c(glob[:, 3]), off=off,
                e_ids=c(cat[:, 0].astype(np.uint32)), e_ver=c(cat[:, 1].astype(np.uint8)),
                e_mark=c(cat[:, 2].astype(np.uint32)), e_freq=c(cat[:, 3].astype(np.uint32)),
                e_last=c(cat[:, 4]), cur=np.array([x[1] for x in caches], np.uint32),
                at=np.array([x[2] for x in caches], np.uint64))


class Cache:
    """Mirror of a standalone embdispatch::WorkerCache (cache.hpp:73-240)."""

    def __init__(self, o: Oracle, capacity, policy=0):
        self.o = o
        self.h = C.c_void_p()
        o._check(o.lib.orc_cache_create(int(capacity), int(policy), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_cache_destroy(self.h)
            self.h = None

    def touch(self, id_, latest, now, footprint=1.0):
        self.o._check(self.o.lib.orc_cache_touch(self.h, int(id_), int(bool(latest)), int(now),
                                                 float(footprint)))

    def set_version(self, id_, latest):
        self.o._check(self.o.lib.orc_cache_set_version(self.h, int(id_), int(bool(latest))))

    def erase(self, id_):
        self.o._check(self.o.lib.orc_cache_erase(self.h, int(id_)))

    def select_victim(self):
        v = C.c_uint32()
        self.o._check(self.o.lib.orc_cache_select_victim(self.h, C.byref(v)))
        return v.value

    def evict_for(self, needed, pinned=()):
        pins = np.array(sorted(int(x) for x in pinned), np.uint32)
        out = np.empty(max(int(needed), 1) + 1, np.uint32)
        cnt = C.c_uint64()
        self.o._check(self.o.lib.orc_cache_evict_for(self.h, int(needed), _p(pins, C.c_uint32),
                                                     len(pins), _p(out, C.c_uint32),
                                                     C.byref(cnt)))
        return [int(x) for x in out[:cnt.value]]

    def info(self):
        size, mark = C.c_uint64(), C.c_uint32()
        self.o.lib.orc_cache_info(self.h, C.byref(size), C.byref(mark))
        return size.value, mark.value

    def entries(self):
        """(id, version, mark, freq, last_access) rows sorted by id."""
        k = self.info()[0]
        ids, ver = np.empty(k, np.uint32), np.empty(k, np.uint8)
        mk, fq, la = np.empty(k, np.uint32), np.empty(k, np.uint32), np.empty(k, np.uint64)
        self.o.lib.orc_cache_export(self.h, _p(ids, C.c_uint32), _p(ver, C.c_uint8),
                                    _p(mk, C.c_uint32), _p(fq, C.c_uint32), _p(la, C.c_uint64))
        return [(int(ids[t]), int(ver[t]), int(mk[t]), int(fq[t]), int(la[t])) for t in range(k)]


class Sim:
    """Mirror of embdispatch::SimState over the orc_* ABI."""

    def __init__(self, o: Oracle, cfg: Cfg):
        self.o, self.cfg = o, cfg
        self.h = C.c_void_p()
        o._check(o.lib.orc_sim_create(C.byref(cfg.c()), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_sim_destroy(self.h)
            self.h = None

    def build_matrix(self, ids, offsets):
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        out = np.empty(R * self.cfg.n, np.float64)
        self.o._check(self.o.lib.orc_sim_build_matrix(self.h, _p(ids, C.c_uint32),
                                                      _p(offsets, C.c_uint64), R,
                                                      _p(out, C.c_double)))
        return out.reshape(R, self.cfg.n)

    def hitgreedy(self, ids, offsets):
        """baseline_hitgreedy on this simulator's live state."""
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        dec = np.empty(max(R, 1), np.int32)
        self.o._check(self.o.lib.orc_sim_hitgreedy(self.h, _p(ids, C.c_uint32),
                                                   _p(offsets, C.c_uint64), R,
                                                   _p(dec, C.c_int32)))
        return dec[:R]

    def step(self, ids, offsets, decision):
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        dec = np.ascontiguousarray(decision, np.int32)
        rep = Report(self.cfg.n)
        self.o._check(self.o.lib.orc_sim_step(self.h, _p(ids, C.c_uint32),
                                              _p(offsets, C.c_uint64), len(offsets) - 1,
                                              _p(dec, C.c_int32), C.byref(rep.c)))
        return rep.as_dict()

    def iteration(self, ids, offsets, threads=1):
        """Reference run() body; returns (decision, expected_cost, report, times_s)."""
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        dec = np.empty(R, np.int32)
        exp = C.c_double()
        rep = Report(self.cfg.n)
        times = np.zeros(4, np.float64)
        self.o._check(self.o.lib.orc_ref_iteration(self.h, _p(ids, C.c_uint32),
                                                   _p(offsets, C.c_uint64), R, threads,
                                                   _p(dec, C.c_int32), C.byref(exp),
                                                   C.byref(rep.c), _p(times, C.c_double)))
        return dec, exp.value, rep.as_dict(), times

    def seed_entry(self, id_, worker, latest, owner):
        self.o._check(self.o.lib.orc_sim_seed_entry(self.h, id_, worker, int(latest), int(owner)))

    def validate_consistency(self):
        self.o._check(self.o.lib.orc_sim_validate_consistency(self.h))

    def clock(self):
        return int(self.o.lib.orc_sim_clock(self.h))

    def import_state(self, state, clock):
        """Replace the whole state with `state` in canonical_state()'s format
        (global rows [id, owners, latest, resident]; per worker (entries
        [id, version, mark, freq, last_access], current_mark, at_current_mark))."""
        args = state_arrays(state, self.cfg.n)
        self.o._check(self.o.lib.orc_sim_import_state(
            self.h, int(clock), len(args["g_ids"]), _p(args["g_ids"], C.c_uint32),
            _p(args["g_owners"], C.c_uint64), _p(args["g_latest"], C.c_uint64),
            _p(args["g_resident"], C.c_uint64), _p(args["off"], C.c_uint64),
            _p(args["e_ids"], C.c_uint32), _p(args["e_ver"], C.c_uint8),
            _p(args["e_mark"], C.c_uint32), _p(args["e_freq"], C.c_uint32),
            _p(args["e_last"], C.c_uint64), _p(args["cur"], C.c_uint32),
            _p(args["at"], C.c_uint64)))

    def canonical_state(self):
        """Non-zero global masks and per-worker entries, both sorted by id."""
        L = self.o.lib
        cnt = int(L.orc_sim_global_count(self.h))
        ids = np.empty(cnt, np.uint32)
        ow, la, re = (np.empty(cnt, np.uint64) for _ in range(3))
        L.orc_sim_export_global(self.h, _p(ids, C.c_uint32), _p(ow, C.c_uint64),
                                _p(la, C.c_uint64), _p(re, C.c_uint64))
        keep = (ow | la | re) != 0
        order = np.argsort(ids[keep], kind="stable")
        glob = np.stack([ids[keep].astype(np.uint64), ow[keep], la[keep], re[keep]], 1)[order]
        caches = []
        for j in range(self.cfg.n):
            sz = int(L.orc_sim_cache_size(self.h, j))
            cid = np.empty(sz, np.uint32)
            ver = np.empty(sz, np.uint8)
            mk = np.empty(sz, np.uint32)
            fq = np.empty(sz, np.uint32)
            la_ = np.empty(sz, np.uint64)
            L.orc_sim_export_cache(self.h, j, _p(cid, C.c_uint32), _p(ver, C.c_uint8),
                                   _p(mk, C.c_uint32), _p(fq, C.c_uint32), _p(la_, C.c_uint64))
            cur = C.c_uint32()
            at = C.c_uint64()
            L.orc_sim_cache_marks(self.h, j, C.byref(cur), C.byref(at))
            o = np.argsort(cid, kind="stable")
            ent = np.stack([cid.astype(np.uint64), ver.astype(np.uint64), mk.astype(np.uint64),
                            fq.astype(np.uint64), la_], 1)[o]
            caches.append((ent, int(cur.value), int(at.value)))
        return glob, caches
