"""B200-native embedding-sample dispatch path (arXiv 2512.21615, `embdispatch`).

Host-side mirror of the reference's C++ API (/root/reference/proj/include/
embdispatch/{types,cost,assign,sim,workload}.hpp) over the C ABI of libedx.so
(include/edx.h).  Names, argument meaning and error classes follow the
reference so parity tests read like its own tests:

    reference (C++)                      here (Python)
    ClusterConfig            types.hpp:71  ClusterConfig
    validate / unit_cost     types.hpp:87  validate / unit_cost
    make_sample              types.hpp:46  make_sample
    Snapshot                  cost.hpp:39  Snapshot (dict id -> EmbeddingState)
    build_matrix             cost.hpp:105  build_matrix  -> CostMatrix
    row_gap_key / rows_by_gap              row_gap_key / rows_by_gap
    hungarian              assign.hpp:80   hungarian     -> AssignmentResult
    greedy_dispatch        assign.hpp:162  greedy_dispatch
    expand_columns         assign.hpp:223  expand_columns
    ecomix                 assign.hpp:247  ecomix        -> DispatchDecision
    decision_cost          assign.hpp:288  decision_cost
    SimState                  sim.hpp:54   SimState (state resident on the GPU)
    ZipfStream           workload.hpp:94   ZipfStream
    TraceSchema/load_schema   :137-172    TraceSchema / load_schema
    TraceStream          workload.hpp:176  TraceStream (CSR batches)

std::invalid_argument -> InvalidArgument (a ValueError), std::logic_error ->
LogicError.  Every computation runs in the CUDA kernels of libedx.so; this
module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence

import numpy as np

from ._lib import (EDX_NUM_PHASES, ClusterConfigC, CudaError, EdxError, EdxRuntimeError,
                   EngineOptionsC, InvalidArgument, LogicError, ReportC, check, lib)

__all__ = [
    "ClusterConfig", "EmbeddingState", "Snapshot", "CostMatrix", "SquareCost", "AssignmentResult",
    "DispatchDecision", "IterationReport", "SimState", "ZipfStream",
    "TraceSchema", "load_schema", "TraceStream", "validate", "unit_cost",
    "make_sample", "to_csr", "build_matrix", "expected_cost", "row_gap_key", "rows_by_gap", "hungarian",
    "hungarian_blocks", "greedy_dispatch", "expand_columns", "ecomix", "decision_cost",
    "exact_multiplicity", "InvalidArgument", "LogicError", "EdxRuntimeError", "CudaError",
    "EdxError", "EDX_NUM_PHASES", "WorkerCache", "VictimPolicy", "CacheEntry",
]

_P = C.POINTER


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(_P(t))


# ------------------------------------------------------------------- types
@dataclass
class ClusterConfig:
    """embdispatch::ClusterConfig (types.hpp:71-82)."""
    n: int = 8
    m: int = 128
    bandwidths_bps: Sequence[float] = field(default_factory=list)
    d_tran_bytes: int = 2048
    cache_capacity: int = 0
    alpha: float = 1.0

    def samples_per_iteration(self) -> int:
        return self.n * self.m

    def _c(self):
        bw = np.ascontiguousarray(np.asarray(self.bandwidths_bps, dtype=np.float64))
        self._bw_keep = bw  # keep alive for the call
        return ClusterConfigC(int(self.n), int(self.m), _ptr(bw, C.c_double), len(bw), 0,
                              int(self.d_tran_bytes), int(self.cache_capacity), float(self.alpha))


@dataclass
class EmbeddingState:
    """embdispatch::EmbeddingState (types.hpp:139-156)."""
    owners: int = 0
    latest: int = 0
    resident: int = 0

    def owned_by(self, w): return bool((self.owners >> w) & 1)
    def latest_on(self, w): return bool((self.latest >> w) & 1)
    def resident_on(self, w): return bool((self.resident >> w) & 1)


class Snapshot(dict):
    """embdispatch::Snapshot (cost.hpp:39-48): id -> EmbeddingState."""

    def state_of(self, id_):
        return self.get(int(id_), EmbeddingState())


@dataclass
class CostMatrix:
    """embdispatch::CostMatrix (cost.hpp:52-60); values is rows x cols float64."""
    values: np.ndarray
    row_ids: Optional[np.ndarray] = None

    @property
    def rows(self): return self.values.shape[0]

    @property
    def cols(self): return self.values.shape[1]

    def at(self, r, c): return float(self.values[r, c])


@dataclass
class SquareCost:
    """embdispatch::SquareCost (assign.hpp:62-68)."""
    values: np.ndarray
    col_to_worker: Optional[np.ndarray] = None

    @property
    def order(self): return self.values.shape[0]


@dataclass
class AssignmentResult:
    col_of_row: np.ndarray
    total_cost: float


@dataclass
class DispatchDecision:
    """embdispatch::DispatchDecision (assign.hpp:38-58)."""
    worker_of_sample: np.ndarray

    def validate(self, cfg: ClusterConfig):
        w = np.asarray(self.worker_of_sample)
        if len(w) != cfg.samples_per_iteration():
            raise InvalidArgument("decision does not cover m*n samples")
        if len(w) and (w.min() < 0 or w.max() >= cfg.n):
            raise InvalidArgument("worker id out of range")
        load = np.bincount(w, minlength=cfg.n)
        for j in range(cfg.n):
            if load[j] != cfg.m:
                raise InvalidArgument(f"worker {j} received {load[j]} samples, expected {cfg.m}")


@dataclass
class IterationReport:
    """embdispatch::IterationReport (sim.hpp:38-50)."""
    iteration: int
    miss_pull_w: List[int]
    update_push_w: List[int]
    evict_push_w: List[int]
    cost_w: List[float]
    miss_pull: int
    update_push: int
    evict_push: int
    cost_s: float
    hits: int
    lookups: int
    expected_cost_s: float = 0.0
    has_expected: bool = False

    def as_dict(self):
        return dict(iteration=self.iteration, miss_pull=self.miss_pull,
                    update_push=self.update_push, evict_push=self.evict_push, hits=self.hits,
                    lookups=self.lookups, cost_s=self.cost_s, miss_pull_w=list(self.miss_pull_w),
                    update_push_w=list(self.update_push_w), evict_push_w=list(self.evict_push_w),
                    cost_w=list(self.cost_w))


class _Report:
    def __init__(self, n):
        self.mp = np.zeros(n, np.uint64)
        self.up = np.zeros(n, np.uint64)
        self.ep = np.zeros(n, np.uint64)
        self.cw = np.zeros(n, np.float64)
        self.c = ReportC(0, 0, 0, 0, 0, 0, 0.0, _ptr(self.mp, C.c_uint64), _ptr(self.up, C.c_uint64),
                         _ptr(self.ep, C.c_uint64), _ptr(self.cw, C.c_double))

    def result(self) -> IterationReport:
        c = self.c
        return IterationReport(int(c.iteration), [int(x) for x in self.mp], [int(x) for x in self.up],
                               [int(x) for x in self.ep], [float(x) for x in self.cw],
                               int(c.miss_pull), int(c.update_push), int(c.evict_push),
                               float(c.cost_s), int(c.hits), int(c.lookups))


# ------------------------------------------------------------ free functions
def validate(cfg: ClusterConfig, max_sample_len: int) -> None:
    """validate(ClusterConfig, max_sample_len) — types.hpp:87-108."""
    c = cfg._c()
    check(lib().edx_validate_config(C.byref(c), int(max_sample_len)))


def unit_cost(cfg: ClusterConfig, worker: int) -> float:
    """unit_cost(cfg, worker).seconds — types.hpp:112-120."""
    if worker < 0 or worker >= cfg.n or worker >= len(cfg.bandwidths_bps):
        raise InvalidArgument(f"worker id {worker} out of range")
    out = np.empty(cfg.n, np.float64)
    c = cfg._c()
    check(lib().edx_unit_costs(C.byref(c), _ptr(out, C.c_double)))
    return float(out[worker])


def make_sample(raw_ids: Iterable[int]) -> List[int]:
    """make_sample — types.hpp:46-60: dedupe, first occurrence wins."""
    raw = list(raw_ids)
    if not raw:
        raise InvalidArgument("embedding sample must contain at least one id")
    seen, out = set(), []
    for x in raw:
        if x not in seen:
            seen.add(x)
            out.append(int(x))
    return out


def to_csr(samples) -> tuple:
    """samples (list of id lists, or an (ids, offsets) pair) -> (ids u32, offsets u64)."""
    if isinstance(samples, tuple) and len(samples) == 2:
        ids, offs = samples
        return (np.ascontiguousarray(ids, np.uint32), np.ascontiguousarray(offs, np.uint64))
    lens = [len(s) for s in samples]
    offs = np.zeros(len(samples) + 1, np.uint64)
    offs[1:] = np.cumsum(lens)
    ids = np.fromiter((x for s in samples for x in s), dtype=np.uint32, count=int(offs[-1]))
    return ids, offs


def _snapshot_arrays(snap):
    keys = np.array(sorted(int(k) for k in snap), np.uint32) if snap else np.zeros(0, np.uint32)
    ow = np.array([snap[int(k)].owners for k in keys], np.uint64)
    la = np.array([snap[int(k)].latest for k in keys], np.uint64)
    re = np.array([snap[int(k)].resident for k in keys], np.uint64)
    return keys, ow, la, re


def _sizes_of(ids, size_of):
    """SizeLookupFn (cost.hpp:64) evaluated once per id position, in order."""
    return np.fromiter((int(size_of(int(x))) for x in ids), dtype=np.uint64, count=len(ids))


def build_matrix(samples, snap, cfg: ClusterConfig, size_of=None) -> CostMatrix:
    """build_matrix — cost.hpp:105-125.  `snap` is a Snapshot or a SimState
    snapshot view; `size_of` (optional) maps an id to its transfer size in
    bytes (SizeLookupFn, cost.hpp:64-73) instead of the uniform d_tran."""
    if isinstance(snap, _EngineSnapshot):
        if size_of is None:
            return snap.engine._build_view(samples)
        snap = snap.engine.snapshot_dict()
    ids, offs = to_csr(samples)
    R = len(offs) - 1
    keys, ow, la, re = _snapshot_arrays(snap or {})
    out = np.empty((max(R, 0), cfg.n), np.float64)
    c = cfg._c()
    if size_of is None:
        check(lib().edx_build_matrix(C.byref(c), _ptr(keys, C.c_uint32), _ptr(ow, C.c_uint64),
                                     _ptr(la, C.c_uint64), _ptr(re, C.c_uint64), len(keys),
                                     _ptr(ids, C.c_uint32), _ptr(offs, C.c_uint64), R,
                                     _ptr(out, C.c_double)))
    else:
        sz = _sizes_of(ids, size_of)
        check(lib().edx_build_matrix_sized(C.byref(c), _ptr(keys, C.c_uint32), _ptr(ow, C.c_uint64),
                                           _ptr(la, C.c_uint64), len(keys), _ptr(ids, C.c_uint32),
                                           _ptr(offs, C.c_uint64), R, _ptr(sz, C.c_uint64),
                                           _ptr(out, C.c_double)))
    return CostMatrix(out, np.arange(R, dtype=np.uint64))


def expected_cost(sample, worker: int, snap, cfg: ClusterConfig, size_of=None) -> float:
    """expected_cost — cost.hpp:81-100 (one cell, optional SizeLookupFn)."""
    if not 0 <= int(worker) < cfg.n:
        raise InvalidArgument("worker id out of range")
    if isinstance(snap, _EngineSnapshot):
        snap = snap.engine.snapshot_dict()
    ids, offs = to_csr([sample])
    keys, ow, la, _ = _snapshot_arrays(snap or {})
    row = np.empty(cfg.n, np.float64)
    c = cfg._c()
    if size_of is None:
        check(lib().edx_expected_costs(C.byref(c), _ptr(keys, C.c_uint32), _ptr(ow, C.c_uint64),
                                       _ptr(la, C.c_uint64), len(keys), _ptr(ids, C.c_uint32),
                                       _ptr(offs, C.c_uint64), 1, _ptr(row, C.c_double)))
    else:
        sz = _sizes_of(ids, size_of)
        check(lib().edx_expected_costs_sized(C.byref(c), _ptr(keys, C.c_uint32),
                                             _ptr(ow, C.c_uint64), _ptr(la, C.c_uint64),
                                             len(keys), _ptr(ids, C.c_uint32),
                                             _ptr(offs, C.c_uint64), 1, _ptr(sz, C.c_uint64),
                                             _ptr(row, C.c_double)))
    return float(row[int(worker)])


def _vals(matrix):
    v = matrix.values if isinstance(matrix, (CostMatrix, SquareCost)) else matrix
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    if v.ndim == 1:
        v = v.reshape(1, -1)
    return v


def row_gap_key(matrix, row: int) -> float:
    """row_gap_key — cost.hpp:130-146."""
    v = _vals(matrix)
    out = C.c_double()
    check(lib().edx_row_gap_key(v.shape[0], v.shape[1], _ptr(v, C.c_double), int(row), C.byref(out)))
    return out.value


def rows_by_gap(matrix) -> np.ndarray:
    """rows_by_gap — assign.hpp:197-207."""
    v = _vals(matrix)
    out = np.empty(v.shape[0], np.uint64)
    check(lib().edx_rows_by_gap(v.shape[0], v.shape[1], _ptr(v, C.c_double), _ptr(out, C.c_uint64)))
    return out


def hungarian(sq) -> AssignmentResult:
    """hungarian(const SquareCost&) — assign.hpp:80-157."""
    v = np.ascontiguousarray(np.asarray(sq.values if isinstance(sq, SquareCost) else sq,
                                        dtype=np.float64))
    if v.ndim != 2 or v.shape[0] != v.shape[1]:
        k = v.shape[0] if v.ndim >= 1 else 0
        if k == 0:
            raise InvalidArgument("solver needs at least one row")
        raise InvalidArgument("cost matrix must be square")
    k = v.shape[0]
    if k < 1:
        raise InvalidArgument("solver needs at least one row")
    cols = np.empty(k, np.uint64)
    total = C.c_double()
    check(lib().edx_hungarian(k, _ptr(v, C.c_double), _ptr(cols, C.c_uint64), C.byref(total)))
    return AssignmentResult(cols, total.value)


def hungarian_blocks(matrix, block_rows, mult: int) -> AssignmentResult:
    """hungarian(expand_columns(matrix, block_rows, mult)) without materialising
    the column-expanded k x k matrix (assign.hpp:223-241, 80-157)."""
    v = _vals(matrix)
    rows = np.ascontiguousarray(block_rows, np.uint64)
    k = v.shape[1] * int(mult)
    if len(rows) != k:
        raise InvalidArgument("row count must equal cols * multiplicity")
    cols = np.empty(k, np.uint64)
    total = C.c_double()
    check(lib().edx_hungarian_blocks(v.shape[0], v.shape[1], _ptr(v, C.c_double),
                                     _ptr(rows, C.c_uint64), int(mult), _ptr(cols, C.c_uint64),
                                     C.byref(total)))
    return AssignmentResult(cols, total.value)


def greedy_dispatch(matrix, rows, capacity):
    """greedy_dispatch — assign.hpp:162-192; returns [(row, worker), ...]."""
    v = _vals(matrix)
    order = np.ascontiguousarray(rows, np.uint64)
    cap = np.ascontiguousarray(capacity, np.int32)
    if len(cap) != v.shape[1]:
        raise InvalidArgument("need one capacity per worker")
    out_r = np.empty(len(order), np.uint64)
    out_w = np.empty(len(order), np.int32)
    check(lib().edx_greedy_dispatch(v.shape[0], v.shape[1], _ptr(v, C.c_double),
                                    _ptr(order, C.c_uint64), len(order), _ptr(cap, C.c_int32),
                                    _ptr(out_r, C.c_uint64), _ptr(out_w, C.c_int32)))
    return [(int(r), int(w)) for r, w in zip(out_r, out_w)]


def exact_multiplicity(m: int, alpha: float) -> int:
    """detail::exact_multiplicity — assign.hpp:213-216."""
    import math
    return max(0, min(int(math.floor(m * alpha + 1e-9)), m))


def expand_columns(matrix, rows, mult: int) -> SquareCost:
    """expand_columns — assign.hpp:223-241 (host-side view, for API parity; the
    device solver never materialises it, see hungarian_blocks)."""
    v = _vals(matrix)
    rows = np.asarray(rows, np.int64)
    k = len(rows)
    if k != v.shape[1] * int(mult):
        raise InvalidArgument("row count must equal cols * multiplicity")
    col_to_worker = (np.arange(k) // max(int(mult), 1)).astype(np.int32)
    return SquareCost(v[rows][:, col_to_worker].copy(), col_to_worker)


def ecomix(matrix, cfg: ClusterConfig) -> DispatchDecision:
    """ecomix — assign.hpp:247-285."""
    if isinstance(matrix, _EngineMatrix):
        return matrix.engine._dispatch_view(cfg.alpha)
    v = _vals(matrix)
    rid = None
    if isinstance(matrix, CostMatrix) and matrix.row_ids is not None:
        rid = np.ascontiguousarray(matrix.row_ids, np.uint64)
    dec = np.empty(v.shape[0], np.int32)
    c = cfg._c()
    check(lib().edx_ecomix(C.byref(c), v.shape[0], v.shape[1], _ptr(v, C.c_double),
                           _ptr(rid, C.c_uint64), _ptr(dec, C.c_int32)))
    return DispatchDecision(dec)


def baseline_hitgreedy(samples, snap, cfg: ClusterConfig) -> DispatchDecision:
    """baseline_hitgreedy — assign.hpp:346-392 (relevance-score baseline): each
    sample scores a worker by its ids' latest copies there; strongest affinity
    commits first; ties to the least-loaded, then lowest-indexed worker.
    `snap` is a Snapshot or a SimState snapshot view (the engine's live state)."""
    if isinstance(snap, _EngineSnapshot):
        return snap.engine._hitgreedy_view(samples)
    ids, offs = to_csr(samples)
    R = len(offs) - 1
    keys, ow, la, _ = _snapshot_arrays(snap or {})
    dec = np.empty(max(R, 1), np.int32)
    c = cfg._c()
    check(lib().edx_hitgreedy(C.byref(c), _ptr(keys, C.c_uint32), _ptr(ow, C.c_uint64),
                              _ptr(la, C.c_uint64), len(keys), _ptr(ids, C.c_uint32),
                              _ptr(offs, C.c_uint64), R, _ptr(dec, C.c_int32)))
    return DispatchDecision(dec[:R])


def decision_cost(matrix, decision) -> float:
    """decision_cost — assign.hpp:288-298."""
    v = _vals(matrix)
    d = np.ascontiguousarray(decision.worker_of_sample if isinstance(decision, DispatchDecision)
                             else decision, np.int32)
    if len(d) != v.shape[0]:
        raise InvalidArgument("decision and matrix disagree on sample count")
    out = C.c_double()
    check(lib().edx_decision_cost(v.shape[0], v.shape[1], _ptr(v, C.c_double),
                                  _ptr(d, C.c_int32), C.byref(out)))
    return out.value


# ------------------------------------------------------------------- engine
class _EngineSnapshot:
    """SimState::snapshot() (sim.hpp:71-82): a zero-copy view of the live
    device state, valid until the next step."""

    def __init__(self, engine):
        self.engine = engine


class _EngineMatrix(CostMatrix):
    """A CostMatrix whose device copy stays in the engine for ecomix."""

    def __init__(self, values, engine):
        super().__init__(values, np.arange(values.shape[0], dtype=np.uint64))
        self.engine = engine


class SimState:
    """embdispatch::SimState (sim.hpp:54-268) with its global state and per-
    worker caches resident on a B200.

    id_space: > 0 selects the dense fast path (ids in [0, id_space), tables
    indexed by id); 0 accepts any uint32 id through the device id table
    (ids.cu), which grows as new ids arrive.
    max_batch_ids: capacity of one batch's id stream (sum of sample lengths)."""

    def __init__(self, cfg: ClusterConfig, id_space: int = 0, max_batch_ids: int = 1 << 20,
                 device: int = 0,
                 rank: int = 0, world_size: int = 1, nccl_id: Optional[bytes] = None):
        self.cfg = cfg
        self._h = C.c_void_p()
        self._nid = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        opt = EngineOptionsC(int(device), 0, int(id_space), int(max_batch_ids), int(rank),
                             int(world_size),
                             C.cast(self._nid, C.c_void_p) if self._nid is not None else None)
        c = cfg._c()
        check(lib().edx_engine_create(C.byref(c), C.byref(opt), C.byref(self._h)))
        self._batch = None

    def close(self):
        if getattr(self, "_h", None):
            lib().edx_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def clock(self) -> int:
        return int(lib().edx_engine_clock(self._h))

    def stream_handle(self) -> int:
        """The engine's cudaStream_t as an integer (for torch.cuda.ExternalStream)."""
        s = C.c_void_p()
        check(lib().edx_engine_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def snapshot(self):
        return _EngineSnapshot(self)

    def config(self):
        return self.cfg

    # -- batch-level calls
    def load(self, samples, on_device: bool = False, ids_ptr=None, offsets_ptr=None, rows=None,
             total_ids=None):
        """Host samples (CSR or list of id lists), or a device batch by pointer; a
        device batch with `total_ids` given is loaded without a host round trip."""
        if on_device:
            if total_ids is not None:
                check(lib().edx_engine_load_device_batch(self._h, C.c_void_p(ids_ptr),
                                                         C.c_void_p(offsets_ptr), int(rows),
                                                         int(total_ids)))
            else:
                check(lib().edx_engine_load_batch(self._h, C.c_void_p(ids_ptr),
                                                  C.c_void_p(offsets_ptr), int(rows), 1))
            return
        ids, offs = to_csr(samples)
        self._batch = (ids, offs)
        check(lib().edx_engine_load_batch(self._h, ids.ctypes.data_as(C.c_void_p),
                                          offs.ctypes.data_as(C.c_void_p), len(offs) - 1, 0))

    def _build_view(self, samples) -> CostMatrix:
        self.load(samples)
        out = np.empty((len(self._batch[1]) - 1, self.cfg.n), np.float64)
        check(lib().edx_engine_build(self._h, _ptr(out, C.c_double)))
        return _EngineMatrix(out, self)

    def build(self, out: Optional[np.ndarray] = None):
        check(lib().edx_engine_build(self._h, _ptr(out, C.c_double)))
        return out

    def _hitgreedy_view(self, samples) -> DispatchDecision:
        self.load(samples)
        return DispatchDecision(self.dispatch_hitgreedy())

    def _dispatch_view(self, alpha) -> DispatchDecision:
        R = self.cfg.samples_per_iteration()
        dec = np.empty(R, np.int32)
        check(lib().edx_engine_dispatch(self._h, float(alpha), _ptr(dec, C.c_int32), None))
        return DispatchDecision(dec)

    def dispatch(self, alpha: float = -1.0, want_decision=True, want_expected=True):
        R = self.cfg.samples_per_iteration()
        dec = np.empty(R, np.int32) if want_decision else None
        exp = C.c_double()
        check(lib().edx_engine_dispatch(self._h, float(alpha), _ptr(dec, C.c_int32),
                                        C.byref(exp) if want_expected else None))
        return dec, (exp.value if want_expected else None)

    def dispatch_hitgreedy(self, want_decision=True):
        """baseline_hitgreedy (assign.hpp:346-392) on the loaded batch and the live
        state; the decision stays on device for step()."""
        dec = np.empty(self.cfg.samples_per_iteration(), np.int32) if want_decision else None
        check(lib().edx_engine_dispatch_hitgreedy(self._h, _ptr(dec, C.c_int32)))
        return dec

    def step(self, samples=None, decision=None) -> IterationReport:
        """SimState::step(samples, decision) — sim.hpp:87-218.  samples None =
        the batch already loaded; decision None = the engine's last dispatch."""
        if samples is not None:
            self.load(samples)
        d = None
        if decision is not None:
            d = np.ascontiguousarray(decision.worker_of_sample if isinstance(decision, DispatchDecision)
                                     else decision, np.int32)
            if len(d) != self.cfg.samples_per_iteration():
                raise InvalidArgument("decision does not cover m*n samples")
        rep = _Report(self.cfg.n)
        check(lib().edx_engine_step(self._h, _ptr(d, C.c_int32), C.byref(rep.c)))
        return rep.result()

    def iterate(self, ids, offsets, want_decision=True, prefetch_next=None):
        """One run() iteration (sim.hpp:421-441) on host buffers.  With
        prefetch_next=(ids, offsets) the next batch's host->device copy is issued
        once this iteration is launched (edx_engine_iterate_prefetch)."""
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        dec = np.empty(R, np.int32) if want_decision else None
        exp = C.c_double()
        rep = _Report(self.cfg.n)
        if prefetch_next is None:
            check(lib().edx_engine_iterate(self._h, ids.ctypes.data_as(C.c_void_p),
                                           offsets.ctypes.data_as(C.c_void_p), R, 0,
                                           _ptr(dec, C.c_int32), C.byref(exp), C.byref(rep.c)))
        else:
            nids = np.ascontiguousarray(prefetch_next[0], np.uint32)
            noffs = np.ascontiguousarray(prefetch_next[1], np.uint64)
            check(lib().edx_engine_iterate_prefetch(
                self._h, ids.ctypes.data_as(C.c_void_p), offsets.ctypes.data_as(C.c_void_p), R,
                nids.ctypes.data_as(C.c_void_p), noffs.ctypes.data_as(C.c_void_p), len(noffs) - 1,
                _ptr(dec, C.c_int32), C.byref(exp), C.byref(rep.c)))
            self._prefetched = (getattr(self, "_prefetched", ()) + ((nids, noffs),))[-2:]
        r = rep.result()
        r.expected_cost_s, r.has_expected = exp.value, True
        return dec, r

    def prefetch(self, ids, offsets):
        """Start the host->device copy of a host batch on the engine's copy stream
        (edx_engine_prefetch); a later iterate()/load() with the same arrays uses
        it.  Pass pinned arrays for an asynchronous copy; they must stay unchanged
        until that call (the engine keeps a reference to the last two)."""
        ids = np.ascontiguousarray(ids, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        check(lib().edx_engine_prefetch(self._h, ids.ctypes.data_as(C.c_void_p),
                                        offsets.ctypes.data_as(C.c_void_p), len(offsets) - 1))
        self._prefetched = (getattr(self, "_prefetched", ()) + ((ids, offsets),))[-2:]

    def iterate_device(self, ids_ptr, offsets_ptr, rows, total_ids, want_decision=True,
                       want_expected=True):
        """One run() iteration on a batch already in device memory (pointers),
        its id count declared; a CUDA-graph replay when the engine allows it."""
        dec = np.empty(int(rows), np.int32) if want_decision else None
        exp = C.c_double()
        rep = _Report(self.cfg.n)
        check(lib().edx_engine_iterate_device(self._h, C.c_void_p(ids_ptr), C.c_void_p(offsets_ptr),
                                              int(rows), int(total_ids), _ptr(dec, C.c_int32),
                                              C.byref(exp) if want_expected else None,
                                              C.byref(rep.c)))
        r = rep.result()
        if want_expected:
            r.expected_cost_s, r.has_expected = exp.value, True
        return dec, r

    # -- state access (parity / tests)
    def seed_entry(self, id_, worker, latest, owner):
        check(lib().edx_engine_seed_entry(self._h, int(id_), int(worker), int(bool(latest)),
                                          int(bool(owner))))

    def state_of(self, id_) -> EmbeddingState:
        o, l, r = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().edx_engine_state_of(self._h, int(id_), C.byref(o), C.byref(l), C.byref(r)))
        return EmbeddingState(o.value, l.value, r.value)

    def validate_consistency(self):
        check(lib().edx_engine_validate_consistency(self._h))

    def import_snapshot(self, snap):
        keys, ow, la, re = _snapshot_arrays(snap)
        check(lib().edx_engine_import_snapshot(self._h, _ptr(keys, C.c_uint32), _ptr(ow, C.c_uint64),
                                               _ptr(la, C.c_uint64), _ptr(re, C.c_uint64), len(keys)))

    def import_state(self, state, clock):
        """Replace the whole state (edx_engine_import_state) with `state` in
        canonical_state()'s format: global rows [id, owners, latest, resident]
        and per worker (entries [id, version, mark, freq, last_access],
        current_mark, at_current_mark).  The result is validated."""
        glob, caches = state
        glob = np.asarray(glob, np.uint64).reshape(-1, 4)
        n = self.cfg.n
        if len(caches) != n:
            raise InvalidArgument("one cache per worker")
        ents = [np.asarray(c[0], np.uint64).reshape(-1, 5) for c in caches]
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum([len(x) for x in ents])
        cat = np.concatenate(ents) if ents else np.zeros((0, 5), np.uint64)
        cc = np.ascontiguousarray
        g_ids, e_ids = cc(glob[:, 0].astype(np.uint32)), cc(cat[:, 0].astype(np.uint32))
        g_ow, g_la, g_re = cc(glob[:, 1]), cc(glob[:, 2]), cc(glob[:, 3])
        e_ver, e_mk = cc(cat[:, 1].astype(np.uint8)), cc(cat[:, 2].astype(np.uint32))
        e_fq, e_la = cc(cat[:, 3].astype(np.uint32)), cc(cat[:, 4])
        cur = np.array([c[1] for c in caches], np.uint32)
        at = np.array([c[2] for c in caches], np.uint64)
        check(lib().edx_engine_import_state(
            self._h, int(clock), len(g_ids), _ptr(g_ids, C.c_uint32), _ptr(g_ow, C.c_uint64),
            _ptr(g_la, C.c_uint64), _ptr(g_re, C.c_uint64), _ptr(off, C.c_uint64),
            _ptr(e_ids, C.c_uint32), _ptr(e_ver, C.c_uint8), _ptr(e_mk, C.c_uint32),
            _ptr(e_fq, C.c_uint32), _ptr(e_la, C.c_uint64), _ptr(cur, C.c_uint32),
            _ptr(at, C.c_uint64)))

    def cache_entries(self, worker):
        """WorkerCache::entries() of one worker as an (k, 5) uint64 array of
        (id, version, mark, freq, last_access) rows, ascending id."""
        sz = C.c_uint64()
        check(lib().edx_engine_cache_size(self._h, int(worker), C.byref(sz)))
        k = sz.value
        ids = np.empty(k, np.uint32)
        ver = np.empty(k, np.uint8)
        mk = np.empty(k, np.uint32)
        fq = np.empty(k, np.uint32)
        la = np.empty(k, np.uint64)
        check(lib().edx_engine_export_cache(self._h, int(worker), _ptr(ids, C.c_uint32),
                                            _ptr(ver, C.c_uint8), _ptr(mk, C.c_uint32),
                                            _ptr(fq, C.c_uint32), _ptr(la, C.c_uint64)))
        return np.stack([ids.astype(np.uint64), ver.astype(np.uint64), mk.astype(np.uint64),
                         fq.astype(np.uint64), la], 1) if k else np.zeros((0, 5), np.uint64)

    def cache_marks(self, worker):
        cur, at = C.c_uint32(), C.c_uint64()
        check(lib().edx_engine_cache_marks(self._h, int(worker), C.byref(cur), C.byref(at)))
        return int(cur.value), int(at.value)

    def global_masks(self):
        """(ids, owners, latest, resident) of every id with a non-zero state."""
        cnt = C.c_uint64()
        check(lib().edx_engine_export_global(self._h, None, None, None, None, 0, C.byref(cnt)))
        k = cnt.value
        ids = np.empty(k, np.uint32)
        ow, la, re = (np.empty(k, np.uint64) for _ in range(3))
        check(lib().edx_engine_export_global(self._h, _ptr(ids, C.c_uint32), _ptr(ow, C.c_uint64),
                                             _ptr(la, C.c_uint64), _ptr(re, C.c_uint64), k,
                                             C.byref(cnt)))
        return ids, ow, la, re

    def snapshot_dict(self) -> "Snapshot":
        """A host Snapshot (id -> EmbeddingState) of the live device state."""
        ids, ow, la, re = self.global_masks()
        snap = Snapshot()
        for t in range(len(ids)):
            snap[int(ids[t])] = EmbeddingState(int(ow[t]), int(la[t]), int(re[t]))
        return snap

    def canonical_state(self):
        """(global, caches) in the same canonical form as oracle.pyoracle.Sim."""
        cnt = C.c_uint64()
        check(lib().edx_engine_export_global(self._h, None, None, None, None, 0, C.byref(cnt)))
        k = cnt.value
        ids = np.empty(k, np.uint32)
        ow, la, re = (np.empty(k, np.uint64) for _ in range(3))
        check(lib().edx_engine_export_global(self._h, _ptr(ids, C.c_uint32), _ptr(ow, C.c_uint64),
                                             _ptr(la, C.c_uint64), _ptr(re, C.c_uint64), k,
                                             C.byref(cnt)))
        glob = np.stack([ids.astype(np.uint64), ow, la, re], 1) if k else np.zeros((0, 4), np.uint64)
        caches = [(self.cache_entries(j),) + self.cache_marks(j) for j in range(self.cfg.n)]
        return glob, caches

    # -- profiling
    def last_kernels(self) -> dict:
        """Kernels the last cost build / exact solve / greedy launched."""
        b, s, g = C.c_char_p(), C.c_char_p(), C.c_char_p()
        check(lib().edx_engine_last_kernels(self._h, C.byref(b), C.byref(s), C.byref(g)))
        return {"build": (b.value or b"").decode(), "solver": (s.value or b"").decode(),
                "greedy": (g.value or b"").decode()}

    def set_profiling(self, on: bool):
        check(lib().edx_engine_set_profiling(self._h, int(bool(on))))

    def phase_times(self, reset=True):
        ms = np.zeros(EDX_NUM_PHASES, np.float64)
        counts = np.zeros(2, np.uint64)
        check(lib().edx_engine_phase_times(self._h, _ptr(ms, C.c_double), _ptr(counts, C.c_uint64),
                                           int(bool(reset))))
        return ms, counts


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for a multi-GPU SimState group (rank 0)."""
    buf = C.create_string_buffer(128)
    check(lib().edx_nccl_unique_id(buf, 128))
    return buf.raw


def shard_rows(rows: int, world: int):
    """Row shard [lo, hi) of every rank (edx_shard_rows: the cost build's split)."""
    lo = np.empty(max(world, 1), np.uint64)
    hi = np.empty(max(world, 1), np.uint64)
    check(lib().edx_shard_rows(int(rows), int(world), _ptr(lo, C.c_uint64), _ptr(hi, C.c_uint64)))
    return [(int(a), int(b)) for a, b in zip(lo[:world], hi[:world])]


class HostTransport:
    """An edx_transport over three Python callables on host byte buffers:
    send(buf: np.ndarray[uint8], peer), recv(buf, peer) (fills buf in place),
    broadcast(buf, root) (in place).  For driving the engine's multi-rank
    exchange steps (edx_exchange_*) from a host harness, e.g. torch.distributed
    gloo in tests; an exception in a callable fails the exchange call."""

    def __init__(self, send, recv, broadcast):
        from . import _lib as L

        def wrap(fn):
            def cb(_ctx, buf, nbytes, peer):
                try:
                    arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)), (int(nbytes),)) \
                        if nbytes else np.empty(0, np.uint8)
                    fn(arr, int(peer))
                    return 0
                except Exception:  # reported as the exchange call's error
                    return 1
            return cb
        self._fns = (L.SEND_FN(wrap(send)), L.RECV_FN(wrap(recv)), L.BCAST_FN(wrap(broadcast)))
        self.c = L.TransportC(None, *self._fns)


def exchange_gather_rows(transport: HostTransport, matrix: np.ndarray, world: int, rank: int,
                         root: int = 0) -> None:
    """The multi-GPU engine's row gather (edx_exchange_gather_rows) on a host
    matrix: this rank's shard rows are sent to the root, which receives every
    other rank's rows in place."""
    assert matrix.dtype == np.float64 and matrix.flags.c_contiguous and matrix.ndim == 2
    check(lib().edx_exchange_gather_rows(C.byref(transport.c), _ptr(matrix, C.c_double),
                                         matrix.shape[0], matrix.shape[1], world, rank, root))


def exchange_broadcast_decision(transport: HostTransport, decision: np.ndarray,
                                root: int = 0) -> None:
    """The multi-GPU engine's decision broadcast (edx_exchange_broadcast_decision)."""
    assert decision.dtype == np.int32 and decision.flags.c_contiguous
    check(lib().edx_exchange_broadcast_decision(C.byref(transport.c), _ptr(decision, C.c_int32),
                                                decision.size, root))


def solver_stats(engine=None) -> dict:
    """Counters of the last exact solve (edx_solver_stats)."""
    out = np.zeros(8, np.uint64)
    check(lib().edx_solver_stats(engine.handle if engine is not None else None,
                                 _ptr(out, C.c_uint64)))
    keys = ["steps", "step_cycles", "potential_cycles", "augment_cycles", "rekey_cycles",
            "augment_hops", "rekeyed_columns", "total_cycles"]
    return {k: int(v) for k, v in zip(keys, out)}


# ------------------------------------------------------------------ workload
class ZipfStream:
    """ZipfStream (workload.hpp:94-133): m*n samples of `sample_len` distinct
    Zipf(zipf_s) ids per iteration, reproducible from the seed."""

    def __init__(self, total_embeddings, sample_len, zipf_s, iterations, seed,
                 samples_per_iteration):
        self._h = C.c_void_p()
        self.L, self.R = int(sample_len), int(samples_per_iteration)
        check(lib().edx_zipf_create(int(total_embeddings), int(sample_len), float(zipf_s),
                                    int(iterations), int(seed), int(samples_per_iteration),
                                    C.byref(self._h)))

    def next_iteration(self) -> Optional[np.ndarray]:
        ids = np.empty(self.R * self.L, np.uint32)
        if not lib().edx_zipf_next(self._h, _ptr(ids, C.c_uint32)):
            return None
        return ids

    def __iter__(self):
        while True:
            ids = self.next_iteration()
            if ids is None:
                return
            yield ids

    def offsets(self) -> np.ndarray:
        return (np.arange(self.R + 1, dtype=np.uint64) * np.uint64(self.L))

    def reset(self):
        lib().edx_zipf_reset(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().edx_zipf_destroy(self._h)
            self._h = None


@dataclass
class TraceSchema:
    """TraceSchema (workload.hpp:137-150): (name, size) per table; row ids
    flatten into one id space by the cumulative table sizes."""
    tables: List[tuple] = field(default_factory=list)

    def total_embeddings(self) -> int:
        return sum(size for _, size in self.tables)


_WS = b" \t\n\v\f\r"


def load_schema(path: str) -> TraceSchema:
    """load_schema (workload.hpp:152-172): "name size" per line, blank lines
    skipped; `size` read as `istream >> size_t` does (optional sign, decimal
    prefix, < 2**64, '-' wrapping) and must be non-zero."""
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise EdxRuntimeError(f"cannot open schema file: {path}") from None
    import re
    schema = TraceSchema()
    lines = raw.split(b"\n")
    if lines and lines[-1] == b"":
        lines.pop()
    for no, line in enumerate(lines, 1):
        parts = line.lstrip(_WS)
        if not parts:
            continue
        name_end = next((i for i, ch in enumerate(parts) if ch in _WS), len(parts))
        name, rest = parts[:name_end], parts[name_end:].lstrip(_WS)
        mt = re.match(rb"([+-]?)([0-9]+)", rest)
        size = None
        if mt and int(mt.group(2)) < 2 ** 64:
            size = int(mt.group(2))
            if mt.group(1) == b"-":
                size = (-size) % 2 ** 64
        if not size:
            raise EdxRuntimeError(f"{path}:{no}: expected 'table_name size'")
        schema.tables.append((name.decode("latin-1"), size))
    if not schema.tables:
        raise EdxRuntimeError(f"schema file declares no tables: {path}")
    return schema


class TraceStream:
    """TraceStream (workload.hpp:176-268): one sample per line of decimal ids,
    m*n samples per iteration, a trailing partial iteration dropped with a
    warning.  Parsed once by libedx on all host threads; each iteration is the
    engine's CSR batch `(ids uint32, offsets uint64[R+1])`, ready for
    `SimState.load` / `iterate` / `prefetch`."""

    def __init__(self, path: str, cfg: ClusterConfig, schema: Optional[TraceSchema] = None,
                 warnings=None):
        import sys
        self._h = C.c_void_p()
        names = [n.encode("latin-1") for n, _ in (schema.tables if schema else [])]
        sizes = np.array([sz for _, sz in (schema.tables if schema else [])], np.uint64)
        name_arr = (C.c_char_p * max(1, len(names)))(*names)
        no_tables = (C.c_uint64 * 1)()  # a schema without tables is still a schema
        sizes_p = (None if schema is None else
                   _ptr(sizes, C.c_uint64) if len(sizes) else C.cast(no_tables, _P(C.c_uint64)))
        check(lib().edx_trace_load(path.encode(), len(names), sizes_p, name_arr,
                                   cfg.samples_per_iteration(), int(cfg.cache_capacity),
                                   int(cfg.m), C.byref(self._h)))
        it, dropped, mx = C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib().edx_trace_info(self._h, C.byref(it), C.byref(dropped), C.byref(mx), None)
        self._iterations, self._dropped, self._max = it.value, dropped.value, mx.value
        self.R = cfg.samples_per_iteration()
        self._cursor = 0
        out = sys.stderr if warnings is None else warnings
        if self._dropped and out is not False:
            out.write(f"warning: {path}: dropping {self._dropped} trailing sample(s) "
                      "of a partial iteration\n")

    def iterations(self) -> int: return self._iterations
    def dropped_samples(self) -> int: return self._dropped
    def max_sample_len(self) -> int: return self._max

    def batch_csr(self, it: int):
        ids_p, offs_p, n = _P(C.c_uint32)(), _P(C.c_uint64)(), C.c_uint64()
        check(lib().edx_trace_iteration(self._h, int(it), C.byref(ids_p), C.byref(offs_p),
                                        C.byref(n)))
        ids = np.ctypeslib.as_array(ids_p, (n.value,)).copy() if n.value else \
            np.empty(0, np.uint32)
        return ids, np.ctypeslib.as_array(offs_p, (self.R + 1,)).copy()

    def next_iteration(self):
        if self._cursor >= self._iterations:
            return None
        self._cursor += 1
        return self.batch_csr(self._cursor - 1)

    def __iter__(self):
        while True:
            b = self.next_iteration()
            if b is None:
                return
            yield b

    def reset(self):
        self._cursor = 0

    def __del__(self):
        if getattr(self, "_h", None):
            lib().edx_trace_destroy(self._h)
            self._h = None


# ------------------------------------------------------- standalone WorkerCache
class VictimPolicy:
    """embdispatch::VictimPolicy (cache.hpp:68)."""
    MARK_VERSION = 0
    PRIORITY_RATIO = 1


@dataclass
class CacheEntry:
    """embdispatch::CacheEntry (cache.hpp:36-42)."""
    id: int
    version_latest: bool = True
    mark: int = 1
    frequency: int = 1
    last_access: int = 0


class WorkerCache:
    """embdispatch::WorkerCache (cache.hpp:73-240) on the device, driven entry
    by entry (libedx workercache.cu).  `footprint(id) -> float` feeds the
    kPriorityRatio policy; `evict_for` returns [(victim, needs_push(victim))]."""

    def __init__(self, capacity: int, policy: int = VictimPolicy.MARK_VERSION, footprint=None,
                 device: int = 0):
        self._h = None
        h = C.c_void_p()
        check(lib().edx_cache_create(int(capacity), int(policy), int(device), C.byref(h)))
        self._h = h
        self._cap = int(capacity)
        self._footprint = footprint

    def __del__(self):
        if getattr(self, "_h", None):
            lib().edx_cache_destroy(self._h)
            self._h = None

    def _info(self):
        size, mark, at = C.c_uint64(), C.c_uint32(), C.c_uint64()
        check(lib().edx_cache_info(self._h, C.byref(size), C.byref(mark), C.byref(at)))
        return size.value, mark.value, at.value

    def capacity(self): return self._cap
    def size(self): return self._info()[0]
    def full(self): return self.size() == self._cap
    def free_slots(self): return self._cap - self.size()
    def current_mark(self): return self._info()[1]
    def at_current_mark(self): return self._info()[2]
    def resident(self, id_): return self.find(id_) is not None

    def find(self, id_):
        f, v, mk, fq, la = C.c_int(), C.c_int(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib().edx_cache_find(self._h, int(id_), C.byref(f), C.byref(v), C.byref(mk),
                                   C.byref(fq), C.byref(la)))
        if not f.value:
            return None
        return CacheEntry(int(id_), bool(v.value), mk.value, fq.value, la.value)

    def touch(self, id_, latest: bool, now: int):
        fp = float(self._footprint(int(id_))) if self._footprint else 1.0
        check(lib().edx_cache_touch(self._h, int(id_), int(bool(latest)), int(now), fp))

    def set_version(self, id_, latest: bool):
        check(lib().edx_cache_set_version(self._h, int(id_), int(bool(latest))))

    def erase(self, id_):
        check(lib().edx_cache_erase(self._h, int(id_)))

    def select_victim(self) -> int:
        out = C.c_uint32()
        check(lib().edx_cache_select_victim(self._h, C.byref(out)))
        return out.value

    def evict_for(self, needed: int, needs_push=None, pinned=None):
        pins = np.array(sorted(int(x) for x in pinned), np.uint32) if pinned else np.zeros(0, np.uint32)
        out = np.empty(max(self._cap, 1), np.uint32)
        cnt = C.c_uint64()
        check(lib().edx_cache_evict_for(self._h, int(needed), _ptr(pins, C.c_uint32), len(pins),
                                        _ptr(out, C.c_uint32), C.byref(cnt)))
        return [(int(v), bool(needs_push(int(v))) if needs_push else False)
                for v in out[:cnt.value]]

    def entries(self):
        cnt = C.c_uint64()
        check(lib().edx_cache_export(self._h, None, None, None, None, None, 0, C.byref(cnt)))
        k = cnt.value
        ids, ver = np.empty(k, np.uint32), np.empty(k, np.uint8)
        mk, fq, la = np.empty(k, np.uint32), np.empty(k, np.uint32), np.empty(k, np.uint64)
        check(lib().edx_cache_export(self._h, _ptr(ids, C.c_uint32), _ptr(ver, C.c_uint8),
                                     _ptr(mk, C.c_uint32), _ptr(fq, C.c_uint32),
                                     _ptr(la, C.c_uint64), k, C.byref(cnt)))
        return {int(ids[t]): CacheEntry(int(ids[t]), bool(ver[t]), int(mk[t]), int(fq[t]),
                                        int(la[t])) for t in range(k)}
