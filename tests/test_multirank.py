"""N>1 candidate sharding: contiguous candidate ranges per rank, one min-loc
record per rank all-gathered per iteration, lexicographic (smice, index) merge
(parallel.cpp:21-29 split, reduce.cpp:397-404 tie rule).

* CPU: world_size-2 gloo processes replay whole reductions; each rank scores
  only its shard (the oracle's per-candidate scores stand in for the device
  scorer), all-gathers its record over gloo and merges with the product's
  krg_merge_best. The merged decisions must equal the single-rank argmin at
  every iteration.
* GPU: two engine contexts as rank 0/1 of world 2 on the one GPU, each on its
  own host thread, exchanging records through an in-process all-gather; the
  trace must equal the reference golden trace bit for bit.
"""
from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_io as gi
import oracle_check as oc
import paper_2510_19608_b200 as kr


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_iterations(case: str, e_bar: float, obj: str):
    net = oc.OracleNet(gi.path(case, "net.json"))
    res = oc.run(net, oc.read_currents(gi.path(case, "scen.csv"), net.n), e_bar, obj, None, score_iters=10_000)
    sc = res["scores"]
    its = []
    for it in range(1, len(res["s"]) + 1):
        m = sc["iter"] == it
        its.append((sc["s"][m], sc["r"][m], sc["feasible"][m].astype(bool), sc["smice"][m], sc["max_err"][m]))
    return res, its


def _rank_main(rank: int, world: int, port: int, case: str, e_bar: float, obj: str, q) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    try:
        res, its = _oracle_iterations(case, e_bar, obj)
        L = res["max_err"].shape[1]
        picks = []
        for s, r, feas, smice, merr in its:
            C = len(s)
            b, e = kr.shard_range(C, rank, world)
            # local argmin over this rank's range (strict <: first minimum)
            best = -1
            for i in range(b, e):
                if feas[i] and (best < 0 or smice[i] < smice[best]):
                    best = i
            rec = torch.zeros(2 + L, dtype=torch.float64)
            rec[0] = smice[best] if best >= 0 else float("inf")
            rec[1] = float(best)
            if best >= 0:
                rec[2:] = torch.from_numpy(merr[best])
            allrec = [torch.zeros_like(rec) for _ in range(world)]
            dist.all_gather(allrec, rec)
            sm = [float(x[0]) for x in allrec]
            ix = [int(x[1]) for x in allrec]
            w = kr.merge_best(sm, ix)
            picks.append((ix[w], sm[w], allrec[w][2:].numpy().copy()) if w >= 0 else (-1, None, None))
        q.put((rank, picks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,e_bar,obj", [("c1", 1e-3, "magnitude"), ("c1", 1e-4, "magnitude"),
                                            ("m40", 1e-3, "complex")])
def test_gloo_two_rank_sharding_matches_single_rank(case, e_bar, obj):
    if not oc.available():
        pytest.skip("oracle not built")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, case, e_bar, obj, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res, its = _oracle_iterations(case, e_bar, obj)
    assert [a[0] for a in out[0]] == [b[0] for b in out[1]]  # every rank commits the same candidate
    for t, (s, r, feas, smice, merr) in enumerate(its):
        idx, sm, me = out[0][t]
        # single-rank rule: first minimum over all feasible candidates
        want = min((i for i in range(len(s)) if feas[i]), key=lambda i: (smice[i], i))
        assert idx == want, f"iteration {t + 1}"
        assert (s[idx], r[idx]) == (res["s"][t], res["r"][t])
        assert gi.d2h(sm) == gi.d2h(res["smice"][t])
        np.testing.assert_array_equal(me, res["max_err"][t])


@pytest.mark.gpu
@pytest.mark.parametrize("tag,flags", [("mag_1e-3", dict(e_bar=1e-3)), ("complex_1e-3", dict(e_bar=1e-3, objective="complex"))])
def test_two_rank_engine_on_one_gpu_matches_golden(tag, flags):
    world = 2
    hp = kr.HostProblem(str(gi.path("c1", "net.json")), str(gi.path("c1", "scen.csv")))
    ctxs = [kr.Context(hp, device=0) for _ in range(world)]
    bar = threading.Barrier(world)
    slots: list = [None] * world

    def make_fn(rank):
        def fn(data: bytes) -> bytes:
            slots[rank] = data
            bar.wait(timeout=60)
            out = b"".join(slots)
            bar.wait(timeout=60)
            return out
        return fn

    for r, c in enumerate(ctxs):
        c.set_exchange(r, world, make_fn(r))
    results: list = [None] * world
    errors: list = []

    def run(rank):
        try:
            results[rank] = ctxs[rank].run_reduction(kr.ReductionConfig(**flags))
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    rows, final = gi.read_trace("c1", tag)
    for res in results:
        assert [(t.s, t.r, gi.d2h(t.smice)) for t in res.trace] == [(s, r, sm) for s, r, sm, *_ in rows]
        assert [gi.d2h(e) for e in res.model.final_max_err] == final
