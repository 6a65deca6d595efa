"""ctypes front-end to the C oracle (oracle/kronred_oracle.c).

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg as the checker. Inputs are parsed here straight
from the fixture files (network JSON as io.cpp:103-166 reads it, current-mode
scenario CSV as scenario.cpp:142-212 reads it), independently of the product's
own loader.
"""
from __future__ import annotations

import ctypes
import json
import math
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
LIB_PATH = ROOT / "oracle" / "_build" / "libkronred_oracle.so"

_lib = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class _Net(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("phases", _u8p),
        ("slack", ctypes.c_int32),
        ("slack_v", _f64p),
        ("nb", ctypes.c_int32),
        ("from_", _i32p),
        ("to", _i32p),
        ("y", _f64p),
        ("sh_from", _f64p),
        ("sh_to", _f64p),
        ("is_z", _u8p),
    ]


def available() -> bool:
    """True once the oracle library exists; builds it (gcc, ~1 s) if missing."""
    if not LIB_PATH.exists():
        import subprocess

        subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle_c"], check=False,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle oracle_c`")
        L = ctypes.CDLL(str(LIB_PATH))
        L.oracle_solve.argtypes = [ctypes.POINTER(_Net), _f64p, ctypes.c_int32, _f64p]
        L.oracle_run.argtypes = [ctypes.POINTER(_Net), ctypes.c_int32, _f64p, ctypes.c_double,
                                 ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                 _i32p, _i32p, _f64p, _f64p, _i32p, _i32p, _f64p,
                                 ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _i32p, _i32p,
                                 _f64p, _f64p, _i32p]
        L.oracle_kron.argtypes = [ctypes.POINTER(_Net), ctypes.c_int32, _i32p, _i32p, _f64p, _u8p]
        L.oracle_cdiv.argtypes = [_f64p, ctypes.c_int32, _f64p]
        for f in (L.oracle_solve, L.oracle_run, L.oracle_kron):
            f.restype = ctypes.c_int
        L.oracle_cdiv.restype = None
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


_PH = {"a": 1, "b": 2, "c": 4}


class OracleNet:
    """Arrays of a parsed network JSON, kept alive for the ctypes struct."""

    def __init__(self, path):
        d = json.loads(Path(path).read_text())
        nodes = sorted(d["nodes"], key=lambda x: x["id"])
        self.n = len(nodes)
        self.phases = np.zeros(self.n, np.uint8)
        self.slack = -1
        self.slack_v = np.zeros(6)
        for nd in nodes:
            m = 0
            for ch in nd["phases"]:
                m |= _PH[ch]
            self.phases[nd["id"]] = m
            if nd.get("slack", False):
                self.slack = nd["id"]
                if "slack_voltage" in nd:
                    self.slack_v[:] = np.array(nd["slack_voltage"], float).reshape(6)
                else:  # nominal_slack_voltage (network.cpp:32-39)
                    th = 2.0 * math.pi / 3.0
                    self.slack_v[:] = [1.0, 0.0, math.cos(-th), math.sin(-th), math.cos(th), math.sin(th)]
        br = d["branches"]
        self.nb = len(br)
        self.frm = np.array([b["from"] for b in br], np.int32)
        self.to = np.array([b["to"] for b in br], np.int32)
        self.y = np.zeros((self.nb, 18))
        self.sh_from = np.zeros((self.nb, 18))
        self.sh_to = np.zeros((self.nb, 18))
        self.is_z = np.zeros(self.nb, np.uint8)
        for k, b in enumerate(br):
            if "y_block" in b:
                self.y[k] = np.array(b["y_block"], float).reshape(18)
            else:
                self.y[k] = np.array(b["z_block"], float).reshape(18)
                self.is_z[k] = 1
            if "shunt_from" in b:
                self.sh_from[k] = np.array(b["shunt_from"], float).reshape(18)
            if "shunt_to" in b:
                self.sh_to[k] = np.array(b["shunt_to"], float).reshape(18)
        self.s = _Net(self.n, _p(self.phases, _u8p), self.slack, _p(self.slack_v, _f64p), self.nb,
                      _p(self.frm, _i32p), _p(self.to, _i32p), _p(self.y, _f64p),
                      _p(self.sh_from, _f64p), _p(self.sh_to, _f64p), _p(self.is_z, _u8p))


def read_currents(path, n: int) -> np.ndarray:
    """Current-mode scenario CSV -> injections [L][3n][2] in first-seen id order."""
    groups: dict[str, np.ndarray] = {}
    lines = [ln for ln in Path(path).read_text().splitlines() if ln and not ln.startswith("#")]
    hdr = [f.strip() for f in lines[0].split(",")]
    if hdr != ["scenario_id", "node_id", "phase", "i_re", "i_im"]:
        raise ValueError(f"not a current-mode scenario file: {hdr}")
    for ln in lines[1:]:
        f = [x.strip() for x in ln.split(",")]
        g = groups.setdefault(f[0], np.zeros((3 * n, 2)))
        t = 3 * int(float(f[1])) + "abc".index(f[2])
        g[t, 0] += float(f[3])
        g[t, 1] += float(f[4])
    return np.stack(list(groups.values()))


def solve(net: OracleNet, inj: np.ndarray) -> np.ndarray:
    inj = np.ascontiguousarray(inj, dtype=np.float64)
    nrhs = inj.shape[0]
    out = np.zeros((nrhs, 3 * net.n, 2))
    rc = lib().oracle_solve(ctypes.byref(net.s), _p(inj, _f64p), nrhs, _p(out, _f64p))
    if rc != 0:
        raise RuntimeError(f"oracle_solve failed: {rc}")
    return out


def run(net: OracleNet, inj: np.ndarray, e_bar: float, objective: str = "magnitude",
        target: float | None = None, score_iters: int = 0) -> dict:
    inj = np.ascontiguousarray(inj, dtype=np.float64)
    L = inj.shape[0]
    cap = net.n
    s = np.zeros(cap, np.int32)
    r = np.zeros(cap, np.int32)
    sm = np.zeros(cap)
    me = np.zeros((cap, L))
    ns = np.zeros(cap, np.int32)
    nc = np.zeros(cap, np.int32)
    fin = np.zeros(L)
    scap = max(1, score_iters * net.n * 8)
    si = np.zeros(scap, np.int32)
    ss = np.zeros(scap, np.int32)
    sr = np.zeros(scap, np.int32)
    sf = np.zeros(scap, np.int32)
    ssm = np.zeros(scap)
    sme = np.zeros((scap, L))
    nsc = np.zeros(1, np.int32)
    it = lib().oracle_run(ctypes.byref(net.s), L, _p(inj, _f64p), e_bar,
                          1 if objective == "complex" else 0, target if target is not None else 0.0,
                          1 if target is not None else 0, cap, _p(s, _i32p), _p(r, _i32p),
                          _p(sm, _f64p), _p(me, _f64p), _p(ns, _i32p), _p(nc, _i32p),
                          _p(fin, _f64p), score_iters, scap, _p(si, _i32p), _p(ss, _i32p),
                          _p(sr, _i32p), _p(sf, _i32p), _p(ssm, _f64p), _p(sme, _f64p),
                          _p(nsc, _i32p))
    if it < 0:
        raise RuntimeError(f"oracle_run failed: {it}")
    k = int(nsc[0])
    return {
        "s": s[:it], "r": r[:it], "smice": sm[:it], "max_err": me[:it], "nsup": ns[:it],
        "cands": nc[:it], "final": fin,
        "scores": {"iter": si[:k], "s": ss[:k], "r": sr[:k], "feasible": sf[:k],
                   "smice": ssm[:k], "max_err": sme[:k]},
    }


def kron(net: OracleNet, reduce):
    red = np.ascontiguousarray(reduce, dtype=np.int32)
    kept = np.zeros(net.n, np.int32)
    blocks = np.zeros(net.n * net.n * 18)
    present = np.zeros(net.n * net.n, np.uint8)
    nk = lib().oracle_kron(ctypes.byref(net.s), len(red), _p(red, _i32p), _p(kept, _i32p),
                           _p(blocks, _f64p), _p(present, _u8p))
    if nk < 0:
        raise RuntimeError(f"oracle_kron failed: {nk}")
    blocks = blocks[: nk * nk * 18].reshape(nk, nk, 9, 2)
    present = present[: nk * nk].reshape(nk, nk)
    return kept[:nk], blocks, present


def cdiv(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """GCC/libgcc complex division of complex128 arrays."""
    inp = np.ascontiguousarray(np.stack([a.real, a.imag, b.real, b.imag], axis=-1).reshape(-1))
    out = np.zeros(2 * a.size)
    lib().oracle_cdiv(_p(inp, _f64p), a.size, _p(out, _f64p))
    return out[0::2] + 1j * out[1::2]
