"""Seeded synthetic feeders for parity tests (network JSON + current-mode CSV).

Radial by default, optionally meshed (extra chords), with unbalanced laterals
(child phases a subset of the parent's), optional z_block branches and shunts,
and scenario rows on a random subset of loaded phases. Numbers are written with
repr(), so the product's loader and the oracle's parse identical doubles.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

_PH = "abc"


def _mask_str(m: int) -> str:
    return "".join(_PH[p] for p in range(3) if (m >> p) & 1)


def _block(rng, mask: int, scale: float) -> list:
    g = rng.uniform(0.5, 1.5) * scale
    ratio = rng.uniform(1.0, 3.0)
    m = np.zeros((3, 3), complex)
    for i in range(3):
        for j in range(3):
            if not ((mask >> i) & 1 and (mask >> j) & 1):
                continue
            if i == j:
                m[i, j] = complex(g, -ratio * g)
            else:
                m[i, j] = complex(-0.25 * g, 0.4 * ratio * g) * rng.uniform(0.8, 1.2)
    return [[float(z.real), float(z.imag)] for z in m.reshape(9)]


def _zblock(rng, mask: int) -> list:
    r = rng.uniform(0.002, 0.02)
    x = r * rng.uniform(1.0, 3.0)
    m = np.zeros((3, 3), complex)
    for i in range(3):
        for j in range(3):
            if (mask >> i) & 1 and (mask >> j) & 1:
                m[i, j] = complex(r, x) if i == j else complex(0.3 * r, 0.35 * x)
    return [[float(z.real), float(z.imag)] for z in m.reshape(9)]


def feeder(n: int, seed: int, *, mesh: int = 0, zfrac: float = 0.0, shunts: bool = False,
           lateral: float = 0.35, slack: int = 0) -> dict:
    rng = np.random.default_rng(seed)
    order = list(range(n))
    # slack sits at the root; the remaining ids are shuffled along the tree so
    # node ids are not in depth order
    rest = [i for i in order if i != slack]
    rng.shuffle(rest)
    seq = [slack] + rest
    masks = {slack: 7}
    parent = {}
    branches = []
    for k in range(1, n):
        node = seq[k]
        p = seq[int(rng.integers(max(0, k - 6), k))]
        parent[node] = p
        pm = masks[p]
        m = pm
        if rng.random() < lateral:
            present = [q for q in range(3) if (pm >> q) & 1]
            keep = rng.choice(present, size=int(rng.integers(1, len(present) + 1)), replace=False)
            m = int(sum(1 << int(q) for q in keep))
        masks[node] = m
        branches.append((p, node))
    # chords between nodes with a common phase make the graph meshed
    have = {tuple(sorted(b)) for b in branches}
    tries = 0
    while mesh > 0 and tries < 100 * n:
        tries += 1
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        if tuple(sorted((a, b))) in have or (masks[a] & masks[b]) == 0:
            continue
        have.add(tuple(sorted((a, b))))
        branches.append((a, b))
        mesh -= 1
    nodes = []
    for i in range(n):
        nd = {"id": i, "phases": _mask_str(masks[i]), "slack": i == slack}
        if i == slack:
            th = 2.0 * np.pi / 3.0
            nd["slack_voltage"] = [[1.0, 0.0], [float(np.cos(-th)), float(np.sin(-th))],
                                   [float(np.cos(th)), float(np.sin(th))]]
        nodes.append(nd)
    br = []
    for a, b in branches:
        common = masks[a] & masks[b]
        e = {"from": int(a), "to": int(b)}
        if rng.random() < zfrac:
            e["z_block"] = _zblock(rng, common)
        else:
            e["y_block"] = _block(rng, common, rng.uniform(15.0, 150.0))
        if shunts and rng.random() < 0.3:
            sh = np.zeros(9, complex)
            for q in range(3):
                if (masks[a] >> q) & 1:
                    sh[4 * q] = complex(0.0, rng.uniform(1e-4, 1e-3))
            e["shunt_from"] = [[float(z.real), float(z.imag)] for z in sh]
        br.append(e)
    return {"nodes": nodes, "branches": br}


def currents(net: dict, L: int, seed: int, density: float = 0.7, scale: float = 3e-3) -> str:
    rng = np.random.default_rng(seed + 7919)
    rows = ["scenario_id,node_id,phase,i_re,i_im"]
    for sc in range(L):
        # a slack row first: loaders zero it (scenario.cpp:22-30), and it keeps
        # every scenario non-empty even on a slack-only network
        slack = next(nd["id"] for nd in net["nodes"] if nd["slack"])
        rows.append(f"s{sc},{slack},a,0.5,-0.25")
        for nd in net["nodes"]:
            if nd["slack"]:
                continue
            for ch in nd["phases"]:
                if rng.random() > density:
                    continue
                mag = scale * rng.uniform(0.1, 1.0)
                ang = rng.uniform(-np.pi, np.pi)
                rows.append(f"s{sc},{nd['id']},{ch},{float(mag * np.cos(ang))!r},{float(mag * np.sin(ang))!r}")
    return "\n".join(rows) + "\n"


def write_case(dirpath: Path, n: int, seed: int, L: int = 3, **kw) -> tuple[Path, Path]:
    dirpath = Path(dirpath)
    dirpath.mkdir(parents=True, exist_ok=True)
    net = feeder(n, seed, **kw)
    netp = dirpath / "net.json"
    scp = dirpath / "scen.csv"
    netp.write_text(json.dumps(net))
    scp.write_text(currents(net, L, seed))
    return netp, scp
