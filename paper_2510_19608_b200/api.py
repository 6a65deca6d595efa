"""Python mirror of the reference's reduction interface over the C ABI.

Names and argument meanings follow the reference's public C++ API
(/root/reference/proj/include/kronred/reduce.hpp:19-170, kron.hpp:13-49,
radialize.hpp:14-39, scenario.hpp:15-64, io.hpp:20-74); errors raise the
reference's exception types (errors.hpp:10-37). Every numeric operation runs
in libkronred_b200.so on an sm_100a device; importing this module without the
built library fails loudly, and device entry points fail loudly without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libkronred_b200.so"
if os.environ.get("KRONRED_LIB"):  # an alternative build of the same library (tools/ variant sweeps)
    LIB_PATH = Path(os.environ["KRONRED_LIB"])

KRG_OK, KRG_E_VALIDATION, KRG_E_SOLVER, KRG_E_CUDA, KRG_E_INTERNAL = 0, 2, 3, 4, 5
OBJ_MAGNITUDE, OBJ_COMPLEX = 0, 1


class Error(RuntimeError):
    """kronred::Error"""


class ValidationError(Error):
    """kronred::ValidationError (CLI exit 2)"""


class SolverError(Error):
    """kronred::SolverError{smallest_pivot, node} (CLI exit 3)"""

    def __init__(self, msg: str, smallest_pivot: float = 0.0, node: int = -1):
        super().__init__(msg)
        self.smallest_pivot = smallest_pivot
        self.node = node


class CudaError(Error):
    """Device missing or CUDA failure (no CPU fallback exists)."""


class KrgNetwork(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("phases", C.POINTER(C.c_uint8)), ("slack", C.c_int32),
                ("slack_voltage", C.POINTER(C.c_double)), ("n_branches", C.c_int32),
                ("br_from", C.POINTER(C.c_int32)), ("br_to", C.POINTER(C.c_int32)),
                ("y_series", C.POINTER(C.c_double)), ("shunt_from", C.POINTER(C.c_double)),
                ("shunt_to", C.POINTER(C.c_double))]


class KrgScenarios(C.Structure):
    _fields_ = [("n_scenarios", C.c_int32), ("injections", C.POINTER(C.c_double)),
                ("voltages", C.POINTER(C.c_double))]


class KrgConfig(C.Structure):
    _fields_ = [("e_bar", C.c_double), ("objective", C.c_int32), ("has_target", C.c_int32),
                ("target_reduction", C.c_double), ("use_delta", C.c_int32), ("workers", C.c_int32)]


class KrgBest(C.Structure):
    _fields_ = [("smice", C.c_double), ("index", C.c_int64), ("s", C.c_int32), ("r", C.c_int32)]


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
OBSERVER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                          C.POINTER(C.c_double), C.c_int32, C.c_int32, C.c_double)

_lib: Optional[C.CDLL] = None

# (name, restype, argtypes)
_SIGS = [
    ("krg_last_error", C.c_char_p, []),
    ("krg_last_error_pivot", C.c_double, []),
    ("krg_last_error_node", C.c_int32, []),
    ("krg_version", C.c_char_p, []),
    ("krg_host_load", C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    ("krg_host_view", C.c_int, [C.c_void_p, C.POINTER(KrgNetwork), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.POINTER(C.c_double))]),
    ("krg_host_scenario_id", C.c_char_p, [C.c_void_p, C.c_int32]),
    ("krg_host_free", None, [C.c_void_p]),
    ("krg_validate", C.c_int, [C.POINTER(KrgNetwork)]),
    ("krg_enumerate_after", C.c_int64, [C.POINTER(KrgNetwork), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int64]),
    ("krg_shard_range", None, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("krg_merge_best", C.c_int32, [C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32]),
    ("krg_create", C.c_int, [C.POINTER(KrgNetwork), C.POINTER(KrgScenarios), C.c_int32, C.POINTER(C.c_void_p)]),
    ("krg_create_from_host", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("krg_reload_from_host", C.c_int, [C.c_void_p, C.c_void_p]),
    ("krg_destroy", None, [C.c_void_p]),
    ("krg_selftest_cdiv", C.c_int, [C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double), C.c_int32]),
    ("krg_set_exchange", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, EXCHANGE_FN, C.c_void_p]),
    ("krg_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("krg_last_run_device_loop", C.c_int32, [C.c_void_p]),
    ("krg_set_comm", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p]),
    ("krg_launch_count", C.c_int64, [C.c_void_p]),
    ("krg_scenario_voltages", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("krg_run_reduction", C.c_int, [C.c_void_p, C.POINTER(KrgConfig), OBSERVER_FN, C.c_void_p,
                                    C.POINTER(C.c_void_p)]),
    ("krg_solve", C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double)]),
    ("krg_loop_begin", C.c_int, [C.c_void_p, C.POINTER(KrgConfig)]),
    ("krg_loop_candidates", C.c_int64, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int64]),
    ("krg_loop_score_all", C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                                     C.POINTER(C.c_double)]),
    ("krg_loop_best", C.c_int, [C.c_void_p, C.POINTER(KrgBest), C.POINTER(C.c_double)]),
    ("krg_loop_commit", C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    ("krg_zcols", C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int64]),
    ("krg_loop_base", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("krg_kron_reduce", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_void_p)]),
    ("krg_radialize", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    ("krg_result_iterations", C.c_int32, [C.c_void_p]),
    ("krg_result_trace", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_double)]),
    ("krg_result_n_kept", C.c_int32, [C.c_void_p]),
    ("krg_result_n_scenarios", C.c_int32, [C.c_void_p]),
    ("krg_result_kept", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_uint8)]),
    ("krg_result_n_blocks", C.c_int64, [C.c_void_p]),
    ("krg_result_blocks", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    ("krg_result_final_max_err", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("krg_result_n_clusters", C.c_int32, [C.c_void_p]),
    ("krg_result_clusters", C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("krg_result_n_reinserted", C.c_int32, [C.c_void_p]),
    ("krg_result_reinserted", C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    ("krg_result_total_candidates", C.c_int64, [C.c_void_p]),
    ("krg_result_write_reduced_json", C.c_int, [C.c_void_p, C.c_char_p]),
    ("krg_result_write_trace_csv", C.c_int, [C.c_void_p, C.c_char_p, C.c_int32]),
    ("krg_result_free", None, [C.c_void_p]),
    ("krg_set_profile", C.c_int, [C.c_void_p, C.c_int32]),
    ("krg_kernel_stats", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("krg_fp64_probe", C.c_int, [C.c_int32, C.POINTER(C.c_double)]),
    ("krg_result_device_ms", C.c_double, [C.c_void_p]),
    ("krg_validate_report", C.c_int64, [C.c_void_p, C.c_void_p, C.c_int32, C.c_char_p, C.c_int64]),
    ("krg_selftest_sqrt", C.c_int, [C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_int64)]),
]


def lib() -> C.CDLL:
    """The loaded libkronred_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the B200 path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return [s[0] for s in _SIGS]


def _check(status: int) -> None:
    if status == KRG_OK:
        return
    msg = (lib().krg_last_error() or b"").decode(errors="replace")
    if status == KRG_E_VALIDATION:
        raise ValidationError(msg)
    if status == KRG_E_SOLVER:
        raise SolverError(msg, lib().krg_last_error_pivot(), lib().krg_last_error_node())
    if status == KRG_E_CUDA:
        raise CudaError(msg)
    raise Error(msg)


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# inputs


@dataclass
class Network:
    """network.hpp:13-52 as arrays. y_series/shunts are [nb,9] complex128."""
    phases: np.ndarray            # uint8 [n]
    slack: int
    slack_voltage: np.ndarray     # complex128 [3]
    br_from: np.ndarray           # int32 [nb]
    br_to: np.ndarray             # int32 [nb]
    y_series: np.ndarray          # complex128 [nb, 9]
    shunt_from: Optional[np.ndarray] = None
    shunt_to: Optional[np.ndarray] = None

    @property
    def size(self) -> int:
        return int(self.phases.shape[0])

    def _c(self) -> tuple[KrgNetwork, list]:
        keep = [np.ascontiguousarray(self.phases, np.uint8),
                _f64(np.asarray(self.slack_voltage, np.complex128).view(np.float64)),
                np.ascontiguousarray(self.br_from, np.int32), np.ascontiguousarray(self.br_to, np.int32),
                _f64(np.asarray(self.y_series, np.complex128).reshape(-1).view(np.float64))]
        sf = st = None
        if self.shunt_from is not None:
            sf = _f64(np.asarray(self.shunt_from, np.complex128).reshape(-1).view(np.float64))
            keep.append(sf)
        if self.shunt_to is not None:
            st = _f64(np.asarray(self.shunt_to, np.complex128).reshape(-1).view(np.float64))
            keep.append(st)
        net = KrgNetwork(self.size, _p(keep[0], C.c_uint8), int(self.slack), _p(keep[1], C.c_double),
                         int(keep[2].shape[0]), _p(keep[2], C.c_int32), _p(keep[3], C.c_int32),
                         _p(keep[4], C.c_double), _p(sf, C.c_double) if sf is not None else None,
                         _p(st, C.c_double) if st is not None else None)
        return net, keep


@dataclass
class ScenarioLibrary:
    """scenario.hpp:15-33: ids, injections [L,3n] and (optional) voltages [L,3n]."""
    ids: list
    injections: np.ndarray
    voltages: Optional[np.ndarray] = None
    pq: bool = False

    @property
    def size(self) -> int:
        return len(self.ids)


class HostProblem:
    """read_network_json + load_library's CSV parse (host only, no device)."""

    def __init__(self, network_json: str, scenario_csv: Optional[str] = None):
        h = C.c_void_p()
        _check(lib().krg_host_load(str(network_json).encode(), (str(scenario_csv) if scenario_csv else "").encode(),
                                   C.byref(h)))
        self._h = h
        net = KrgNetwork()
        L = C.c_int32()
        pq = C.c_int32()
        data = C.POINTER(C.c_double)()
        _check(lib().krg_host_view(h, C.byref(net), C.byref(L), C.byref(pq), C.byref(data)))
        n, nb = net.n_nodes, net.n_branches

        def arr(ptr, count, dt):
            return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dt).copy() if count else np.zeros(0, dt)

        cplx = lambda ptr, cnt: arr(ptr, 2 * cnt, np.float64).view(np.complex128)
        self.network = Network(arr(net.phases, n, np.uint8), net.slack, cplx(net.slack_voltage, 3),
                               arr(net.br_from, nb, np.int32), arr(net.br_to, nb, np.int32),
                               cplx(net.y_series, 9 * nb).reshape(nb, 9),
                               cplx(net.shunt_from, 9 * nb).reshape(nb, 9), cplx(net.shunt_to, 9 * nb).reshape(nb, 9))
        ids = [lib().krg_host_scenario_id(h, i).decode() for i in range(L.value)]
        vals = cplx(data, 3 * n * L.value).reshape(L.value, 3 * n) if L.value else np.zeros((0, 3 * n), np.complex128)
        self.library = ScenarioLibrary(ids, vals, None, bool(pq.value))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.krg_host_free(self._h)
            self._h = None


def validate(net: Network) -> None:
    """validate_or_throw (network.cpp:192): raises ValidationError."""
    cn, _keep = net._c()
    _check(lib().krg_validate(C.byref(cn)))


def enumerate_after(net: Network, trajectory: Sequence[tuple[int, int]]) -> list[tuple[int, int]]:
    """enumerate_candidates (reduce.cpp:63-73) after committing `trajectory`."""
    cn, _keep = net._c()
    ts = np.array([t[0] for t in trajectory] or [0], np.int32)
    tr = np.array([t[1] for t in trajectory] or [0], np.int32)
    cap = 2 * net.size + 2
    cs = np.zeros(cap, np.int32)
    cr = np.zeros(cap, np.int32)
    cnt = lib().krg_enumerate_after(C.byref(cn), _p(ts, C.c_int32), _p(tr, C.c_int32), len(trajectory),
                                    _p(cs, C.c_int32), _p(cr, C.c_int32), cap)
    if cnt < 0:
        _check(int(-cnt))
    return list(zip(cs[:cnt].tolist(), cr[:cnt].tolist()))


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    b, e = C.c_int64(), C.c_int64()
    lib().krg_shard_range(count, rank, world, C.byref(b), C.byref(e))
    return b.value, e.value


def merge_best(smice: Sequence[float], index: Sequence[int]) -> int:
    s = _f64(smice)
    i = np.ascontiguousarray(index, np.int64)
    return int(lib().krg_merge_best(_p(s, C.c_double), _p(i, C.c_int64), len(s)))


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 makes it, every rank passes it to
    Context.set_comm)."""
    buf = C.create_string_buffer(128)
    _check(lib().krg_nccl_unique_id(buf))
    return buf.raw


def fp64_probe(device: int = -1) -> float:
    """Measured unfused FP64 rate (GFLOP/s) — the roofline peak for the scorer."""
    g = C.c_double()
    _check(lib().krg_fp64_probe(device, C.byref(g)))
    return g.value


def sqrt_selftest(n: int, lo: float, hi: float) -> int:
    """Bit mismatches of the scorer's branch-free sqrt vs IEEE sqrt (device)."""
    m = C.c_int64()
    _check(lib().krg_selftest_sqrt(n, lo, hi, C.byref(m)))
    return m.value


def cdiv_selftest(quads: np.ndarray, on_device: bool) -> np.ndarray:
    q = _f64(quads).reshape(-1, 4)
    out = np.zeros((q.shape[0], 2))
    _check(lib().krg_selftest_cdiv(_p(q, C.c_double), q.shape[0], _p(out, C.c_double), int(on_device)))
    return out


# ---------------------------------------------------------------------------
# configuration and results


@dataclass
class ReductionConfig:
    """reduce.hpp:21-28"""
    e_bar: float = 1e-3
    objective: str = "mag"          # "mag" | "complex"
    target_reduction: Optional[float] = None
    workers: int = 1                # no device meaning (kept for drop-in)
    use_delta: bool = True
    topology_tol: float = 1e-9

    def _c(self) -> KrgConfig:
        return KrgConfig(float(self.e_bar), OBJ_COMPLEX if self.objective == "complex" else OBJ_MAGNITUDE,
                         int(self.target_reduction is not None),
                         float(self.target_reduction if self.target_reduction is not None else 0.0),
                         int(self.use_delta), int(self.workers))


@dataclass
class TraceRow:
    iteration: int
    s: int
    r: int
    smice: float
    max_err: np.ndarray
    supernode_count: int
    candidate_count: int
    wall_ms: float


@dataclass
class ReducedModel:
    """reduce.hpp:141-152"""
    kept_ids: np.ndarray
    kept_phases: np.ndarray
    y_kron: dict                    # (i, j) original ids -> complex [3,3]
    clusters: dict
    reinserted: list
    final_max_err: np.ndarray


class Result:
    """ReductionResult (reduce.hpp:154-158) backed by the C result object."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        L = lib()
        it = L.krg_result_iterations(handle)
        ns = L.krg_result_n_scenarios(handle)
        s = np.zeros(max(it, 1), np.int32)
        r = np.zeros(max(it, 1), np.int32)
        sm = np.zeros(max(it, 1))
        me = np.zeros(max(it * max(ns, 1), 1))
        snc = np.zeros(max(it, 1), np.int32)
        cc = np.zeros(max(it, 1), np.int32)
        wall = np.zeros(max(it, 1))
        _check(L.krg_result_trace(handle, _p(s, C.c_int32), _p(r, C.c_int32), _p(sm, C.c_double),
                                  _p(me, C.c_double), _p(snc, C.c_int32), _p(cc, C.c_int32), _p(wall, C.c_double)))
        me = me[: it * ns].reshape(it, ns) if ns else np.zeros((it, 0))
        # the trace arrives as arrays; the per-row objects are built on first access
        self.trace_arrays = {"s": s[:it], "r": r[:it], "smice": sm[:it], "max_err": me, "supernode_count": snc[:it],
                             "candidate_count": cc[:it], "wall_ms": wall[:it]}
        self._trace = None
        self.total_candidates = int(L.krg_result_total_candidates(handle))
        self.device_ms = float(L.krg_result_device_ms(handle))
        self.model = self._model()

    @property
    def trace(self) -> list:
        if self._trace is None:
            t = self.trace_arrays
            self._trace = [TraceRow(i + 1, int(t["s"][i]), int(t["r"][i]), float(t["smice"][i]), t["max_err"][i],
                                    int(t["supernode_count"][i]), int(t["candidate_count"][i]), float(t["wall_ms"][i]))
                           for i in range(len(t["s"]))]
        return self._trace

    def _model(self) -> ReducedModel:
        L = lib()
        h = self._h
        nk = L.krg_result_n_kept(h)
        ids = np.zeros(max(nk, 1), np.int32)
        ph = np.zeros(max(nk, 1), np.uint8)
        L.krg_result_kept(h, _p(ids, C.c_int32), _p(ph, C.c_uint8))
        nb = L.krg_result_n_blocks(h)
        bi = np.zeros(max(nb, 1), np.int32)
        bj = np.zeros(max(nb, 1), np.int32)
        vals = np.zeros(max(nb, 1) * 18)
        L.krg_result_blocks(h, _p(bi, C.c_int32), _p(bj, C.c_int32), _p(vals, C.c_double))
        blocks = vals.view(np.complex128).reshape(-1, 3, 3)
        y = {(int(bi[k]), int(bj[k])): blocks[k].copy() for k in range(nb)}
        ncl = L.krg_result_n_clusters(h)
        sup = np.zeros(max(ncl, 1), np.int32)
        off = np.zeros(ncl + 1, np.int32)
        mem = np.zeros(max(L.krg_result_n_kept(h), 1) + 1, np.int32)
        # members total <= n; size generously from the trace-independent bound
        total = 1 << 20
        mem = np.zeros(total, np.int32)
        L.krg_result_clusters(h, _p(sup, C.c_int32), _p(off, C.c_int32), _p(mem, C.c_int32))
        clusters = {int(sup[k]): mem[off[k]:off[k + 1]].tolist() for k in range(ncl)}
        nr = L.krg_result_n_reinserted(h)
        rein = np.zeros(max(nr, 1), np.int32)
        L.krg_result_reinserted(h, _p(rein, C.c_int32))
        ns = L.krg_result_n_scenarios(h)
        fe = np.zeros(max(ns, 1))
        L.krg_result_final_max_err(h, _p(fe, C.c_double))
        return ReducedModel(ids[:nk].copy(), ph[:nk].copy(), y, clusters, rein[:nr].tolist(), fe[:ns].copy())

    def write_reduced_json(self, path: str) -> None:
        _check(lib().krg_result_write_reduced_json(self._h, str(path).encode()))

    def write_trace_csv(self, path: str, zero_wall: bool = False) -> None:
        _check(lib().krg_result_write_trace_csv(self._h, str(path).encode(), int(zero_wall)))

    def reduced_json(self) -> str:
        import tempfile
        with tempfile.NamedTemporaryFile("r", suffix=".json") as f:
            self.write_reduced_json(f.name)
            return Path(f.name).read_text()

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.krg_result_free(self._h)
            self._h = None


# ---------------------------------------------------------------------------
# device context


class Context:
    """One device context (krg_ctx): Y, schedules and scenario data resident in HBM."""

    def __init__(self, problem, library: Optional[ScenarioLibrary] = None, device: int = -1):
        h = C.c_void_p()
        if isinstance(problem, HostProblem):
            _check(lib().krg_create_from_host(problem._h, device, C.byref(h)))
            self.ids = problem.library.ids
            self.n = problem.network.size
        else:
            cn, keep = problem._c()
            scen = None
            if library is not None and library.size:
                inj = _f64(np.asarray(library.injections, np.complex128).view(np.float64))
                keep.append(inj)
                vp = None
                if library.voltages is not None:
                    v = _f64(np.asarray(library.voltages, np.complex128).view(np.float64))
                    keep.append(v)
                    vp = _p(v, C.c_double)
                scen = KrgScenarios(library.size, _p(inj, C.c_double), vp)
            _check(lib().krg_create(C.byref(cn), C.byref(scen) if scen is not None else None, device, C.byref(h)))
            self.ids = library.ids if library is not None else []
            self.n = problem.size
        self._h = h
        self._cb = None

    def reload(self, problem: "HostProblem") -> None:
        """krg_reload_from_host: new admittances and scenarios for the same
        network structure, copied host -> device into this context."""
        _check(lib().krg_reload_from_host(self._h, problem._h))
        self.ids = problem.library.ids

    @property
    def L(self) -> int:
        return len(self.ids)

    @property
    def last_run_device_loop(self) -> bool:
        """The last run_reduction ran as the device-resident loop graph."""
        return bool(lib().krg_last_run_device_loop(self._h))

    def launch_count(self) -> int:
        return int(lib().krg_launch_count(self._h))

    def set_profile(self, on: bool) -> None:
        _check(lib().krg_set_profile(self._h, int(on)))

    def kernel_stats(self, which: int) -> dict:
        n, ms, fl, by = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        _check(lib().krg_kernel_stats(self._h, which, C.byref(n), C.byref(ms), C.byref(fl), C.byref(by)))
        return {"launches": n.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}

    def scenario_voltages(self) -> np.ndarray:
        out = np.zeros(self.L * 3 * self.n * 2)
        _check(lib().krg_scenario_voltages(self._h, _p(out, C.c_double)))
        return out.view(np.complex128).reshape(self.L, 3 * self.n)

    def set_exchange(self, rank: int, world: int, fn: Callable[[bytes], bytes]) -> None:
        """fn(send_bytes) -> concatenated bytes of every rank (rank order)."""

        def _cb(_user, send, recv, nbytes):
            try:
                data = fn(C.string_at(send, nbytes))
                C.memmove(recv, data, len(data))
                return 0
            except Exception:  # noqa: BLE001 - reported as a status code
                return 1

        self._cb = EXCHANGE_FN(_cb)
        _check(lib().krg_set_exchange(self._h, rank, world, self._cb, None))

    def set_comm(self, rank: int, world: int, unique_id: bytes) -> None:
        """In-graph multi-GPU exchange (krg_set_comm): collective over the
        `world` ranks, each with its own context on its own GPU."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        _check(lib().krg_set_comm(self._h, rank, world, unique_id))

    def run_reduction(self, cfg: ReductionConfig, observer: Optional[Callable[[TraceRow], None]] = None) -> Result:
        """run_reduction (reduce.cpp:349-451)."""
        c = cfg._c()
        out = C.c_void_p()
        if observer is not None:
            def _obs(_u, it, s, r, smice, me, snc, cc, wall):
                observer(TraceRow(it, s, r, smice, np.ctypeslib.as_array(me, shape=(self.L,)).copy(), snc, cc, wall))
            cb = OBSERVER_FN(_obs)
        else:
            cb = OBSERVER_FN()
        _check(lib().krg_run_reduction(self._h, C.byref(c), cb, None, C.byref(out)))
        return Result(out)

    def solve(self, injections: np.ndarray) -> np.ndarray:
        """AnchoredSolver::solve batched: [nrhs, 3n] complex -> [nrhs, 3n]."""
        inj = np.atleast_2d(np.asarray(injections, np.complex128))
        src = _f64(inj.view(np.float64))
        out = np.zeros_like(src)
        _check(lib().krg_solve(self._h, _p(src, C.c_double), inj.shape[0], _p(out, C.c_double)))
        return out.view(np.complex128).reshape(inj.shape)

    # loop parity hooks -----------------------------------------------------
    def loop_begin(self, cfg: ReductionConfig) -> None:
        c = cfg._c()
        _check(lib().krg_loop_begin(self._h, C.byref(c)))

    def loop_candidates(self) -> list[tuple[int, int]]:
        cap = 2 * self.n + 2
        cs = np.zeros(cap, np.int32)
        cr = np.zeros(cap, np.int32)
        cnt = lib().krg_loop_candidates(self._h, _p(cs, C.c_int32), _p(cr, C.c_int32), cap)
        if cnt < 0:
            _check(int(-cnt))
        self._ncand = int(cnt)
        return list(zip(cs[:cnt].tolist(), cr[:cnt].tolist()))

    def loop_score_all(self):
        C_ = self._ncand
        sm = np.zeros(max(C_, 1))
        fe = np.zeros(max(C_, 1), np.uint8)
        me = np.zeros(max(C_ * self.L, 1))
        _check(lib().krg_loop_score_all(self._h, _p(sm, C.c_double), _p(fe, C.c_uint8), _p(me, C.c_double)))
        return sm[:C_], fe[:C_].astype(bool), me[: C_ * self.L].reshape(C_, self.L)

    def loop_best(self):
        b = KrgBest()
        me = np.zeros(max(self.L, 1))
        _check(lib().krg_loop_best(self._h, C.byref(b), _p(me, C.c_double)))
        return b.index, b.s, b.r, b.smice, me[: self.L]

    def loop_commit(self, s: int, r: int) -> None:
        _check(lib().krg_loop_commit(self._h, s, r))

    def loop_base(self) -> np.ndarray:
        out = np.zeros(self.L * 3 * self.n * 2)
        _check(lib().krg_loop_base(self._h, _p(out, C.c_double)))
        return out.view(np.complex128).reshape(self.L, 3 * self.n)

    def zcols(self, nphi: int) -> np.ndarray:
        out = np.zeros(nphi * nphi * 2)
        _check(lib().krg_zcols(self._h, _p(out, C.c_double), out.size))
        return out.view(np.complex128).reshape(nphi, nphi)  # [column][row]

    def validate_report(self, result: "Result", bins: int = 20) -> str:
        """make_validate_report + write_validate_report (io.cpp:385-416) as a string."""
        n = lib().krg_validate_report(self._h, result._h, bins, None, 0)
        if n < 0:
            _check(int(-n))
        buf = C.create_string_buffer(int(n) + 1)
        _check(0 if lib().krg_validate_report(self._h, result._h, bins, buf, n + 1) >= 0 else 1)
        return buf.value.decode()

    def kron_reduce(self, reduce: Sequence[int]) -> Result:
        red = np.ascontiguousarray(sorted(set(int(x) for x in reduce)) or [0], np.int32)
        out = C.c_void_p()
        _check(lib().krg_kron_reduce(self._h, _p(red, C.c_int32), len(set(reduce)), C.byref(out)))
        return Result(out)

    def radialize(self, result: Result, with_errors: bool = True) -> Result:
        _check(lib().krg_radialize(self._h, result._h, int(with_errors)))
        result.model = result._model()
        return result

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.krg_destroy(self._h)
            self._h = None


def run_reduction(problem, cfg: ReductionConfig, library: Optional[ScenarioLibrary] = None,
                  observer=None, device: int = -1) -> Result:
    """Module-level run_reduction(net, lib, cfg) (reduce.hpp:168-170)."""
    return Context(problem, library, device).run_reduction(cfg, observer)
