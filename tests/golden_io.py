"""Readers for the golden fixtures produced by tests/golden/make_golden.py."""
from __future__ import annotations

import gzip
import json
import shutil
import struct
import tempfile
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def h2d(h: str) -> float:
    return struct.unpack("<d", bytes.fromhex(h)[::-1])[0]


def d2h(x: float) -> str:
    return struct.pack("<d", x)[::-1].hex()


def path(case: str, name: str) -> Path:
    """Path to a fixture; gzipped fixtures are inflated into a temp dir."""
    p = GOLDEN / case / name
    if p.exists():
        return p
    gz = GOLDEN / case / (name + ".gz")
    if not gz.exists():
        raise FileNotFoundError(p)
    out = Path(tempfile.gettempdir()) / "kronred_golden" / case
    out.mkdir(parents=True, exist_ok=True)
    dst = out / name
    if not dst.exists() or dst.stat().st_mtime < gz.stat().st_mtime:
        with gzip.open(gz, "rb") as f, open(dst, "wb") as g:
            shutil.copyfileobj(f, g)
    return dst


def runs(case: str) -> dict:
    return json.loads((GOLDEN / case / "runs.json").read_text())


def read_trace(case: str, tag: str):
    """-> list of (s, r, smice_hex, [maxerr_hex], supernode_count, candidate_count), final [hex]."""
    rows, final = [], []
    for line in path(case, f"trace_{tag}.txt").read_text().splitlines():
        f = line.split()
        if f[0] == "final":
            final = f[1:]
            continue
        rows.append((int(f[1]), int(f[2]), f[3], f[4:-2], int(f[-2]), int(f[-1])))
    return rows, final


def read_scores(case: str, tag: str):
    """-> {iteration: [(s, r, feasible, smice_hex, [maxerr_hex])]}"""
    out: dict[int, list] = {}
    for line in path(case, f"scores_{tag}.txt").read_text().splitlines():
        f = line.split()
        out.setdefault(int(f[0]), []).append((int(f[1]), int(f[2]), f[3] == "1", f[4], f[5:]))
    return out


def read_solve(case: str, name: str = "solve.txt") -> dict[str, np.ndarray]:
    out = {}
    for line in path(case, name).read_text().splitlines():
        f = line.split()
        vals = np.array([h2d(h) for h in f[1:]])
        out[f[0]] = vals[0::2] + 1j * vals[1::2]
    return out


def read_kron(case: str, k: int):
    red = [int(x) for x in path(case, f"kron_{k}.reduce").read_text().split()]
    blocks = {}
    for line in path(case, f"kron_{k}.txt").read_text().splitlines():
        f = line.split()
        vals = np.array([h2d(h) for h in f[2:]])
        blocks[(int(f[0]), int(f[1]))] = (vals[0::2] + 1j * vals[1::2]).reshape(3, 3)
    return red, blocks
