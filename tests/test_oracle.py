"""Pin the C oracle (oracle/kronred_oracle.c) to the reference's golden vectors.

Every fixture under tests/golden/ was written by the UNMODIFIED reference build
(oracle/_ref, tests/golden/make_golden.py). The oracle must reproduce them bit
for bit: anchored solves (solver.cpp:181-186), per-candidate delta scores
(reduce.cpp:194-244), whole trajectories and final errors of run_reduction
(reduce.cpp:349-451) and kron_reduce blocks (kron.cpp:34-46). CPU only.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import golden_io as gi
import oracle_check as oc

pytestmark = pytest.mark.skipif(not oc.available(), reason="oracle not built (make -C oracle oracle_c)")


def _hex(a):
    return [gi.d2h(float(x)) for x in np.ravel(a)]


def _flags(flags):
    eb = float(flags[flags.index("--e-bar") + 1]) if "--e-bar" in flags else 0.0
    obj = flags[flags.index("--objective") + 1] if "--objective" in flags else "magnitude"
    tgt = float(flags[flags.index("--target") + 1]) if "--target" in flags else None
    return eb, obj, tgt


def _load(case):
    net = oc.OracleNet(gi.path(case, "net.json"))
    inj = oc.read_currents(gi.path(case, "scen.csv"), net.n)
    return net, inj


def _check_trace(case, tag, res):
    rows, final = gi.read_trace(case, tag)
    assert len(rows) == len(res["s"])
    for i, (s, r, smice, errs, nsup, ncand) in enumerate(rows):
        assert (s, r) == (res["s"][i], res["r"][i]), f"iteration {i + 1}"
        assert smice == gi.d2h(res["smice"][i]), f"iteration {i + 1} smice"
        assert errs == _hex(res["max_err"][i]), f"iteration {i + 1} max_err"
        assert (nsup, ncand) == (res["nsup"][i], res["cands"][i])
    assert final == _hex(res["final"])


RUNS = [(case, tag) for case in ("c1", "m40", "s24") for tag, info in gi.runs(case).items()
        if not info.get("radialize") and "--use-delta" not in info["flags"]]  # the oracle restates the delta path


@pytest.mark.parametrize("case,tag", RUNS)
def test_trace_matches_reference(case, tag):
    net, inj = _load(case)
    eb, obj, tgt = _flags(gi.runs(case)[tag]["flags"])
    res = oc.run(net, inj, eb, obj, tgt)
    _check_trace(case, tag, res)


@pytest.mark.parametrize("case,tag", [("c1", "mag_1e-3"), ("c1", "complex_1e-3"), ("m40", "mag_1e-3")])
def test_candidate_scores_match_reference(case, tag):
    golden = gi.read_scores(case, tag)
    net, inj = _load(case)
    eb, obj, _ = _flags(gi.runs(case)[tag]["flags"])
    res = oc.run(net, inj, eb, obj, None, score_iters=max(golden))
    sc = res["scores"]
    k = 0
    for it in sorted(golden):
        for s, r, feas, smice, errs in golden[it]:
            assert (sc["iter"][k], sc["s"][k], sc["r"][k]) == (it, s, r)
            assert bool(sc["feasible"][k]) == feas
            assert gi.d2h(sc["smice"][k]) == smice
            assert _hex(sc["max_err"][k]) == errs
            k += 1
    assert k == len(sc["s"])


@pytest.mark.parametrize("case", ["m40", "s24"])
def test_solves_match_reference(case):
    ref = gi.read_solve(case)
    net, inj = _load(case)
    dim = 3 * net.n
    rhs = [np.zeros((dim, 2))]
    tags = ["v0"]
    for key in ref:
        if key.startswith("e"):
            u = np.zeros((dim, 2))
            u[int(key[1:]), 0] = 1.0
            rhs.append(u)
            tags.append(key)
    L = len([k for k in ref if k.startswith("vhat")])
    # scenario voltages: slack rows / absent phases zeroed first (scenario.cpp:22-30)
    for l in range(L):
        x = inj[l].copy()
        for t in range(dim):
            if t // 3 == net.slack or not (net.phases[t // 3] >> (t % 3)) & 1:
                x[t] = 0.0
        rhs.append(x)
        tags.append(f"vhat{l}")
    out = oc.solve(net, np.stack(rhs))
    for tag, v in zip(tags, out):
        want = ref[tag]
        got = v[:, 0] + 1j * v[:, 1]
        assert _hex(got.real) == _hex(want.real), tag
        assert _hex(got.imag) == _hex(want.imag), tag


@pytest.mark.parametrize("case,k", [(c, k) for c in ("c1", "m40") for k in range(3)])
def test_kron_matches_reference(case, k):
    red, blocks = gi.read_kron(case, k)
    net, _ = _load(case)
    kept, got, present = oc.kron(net, red)
    assert list(kept) == [i for i in range(net.n) if i not in set(red)]
    assert int(present.sum()) == len(blocks)
    pos = {int(k): q for q, k in enumerate(kept)}
    for (oi, oj), blk in blocks.items():
        i, j = pos[oi], pos[oj]
        assert present[i, j], (oi, oj)
        g = got[i, j, :, 0] + 1j * got[i, j, :, 1]
        assert _hex(g.real) == _hex(blk.reshape(9).real), (i, j)
        assert _hex(g.imag) == _hex(blk.reshape(9).imag), (i, j)


def test_cdiv_is_gcc_complex_division():
    # smith-style scaling cases that naive (ac+bd)/(c^2+d^2) gets wrong
    a = np.array([1 + 1j, 1e300 + 1e300j, 3 - 4j, 1e-300 + 1j, 0j])
    b = np.array([1e-310 + 1e-310j, 1e300 + 1e-300j, 0.5 + 0.25j, 1e-300 + 1e-300j, 2 + 0j])
    q = oc.cdiv(a, b)
    assert np.all(np.isfinite(q[1:]))
    assert q[2] == pytest.approx((3 - 4j) / (0.5 + 0.25j), rel=1e-15)
    assert q[4] == 0


@pytest.mark.skipif(os.environ.get("KRONRED_SLOW") != "1", reason="C2 oracle run takes ~9 min; KRONRED_SLOW=1")
def test_c2_trace_matches_reference():
    net = oc.OracleNet(gi.path("c2", "net.json"))
    inj = oc.read_currents(gi.path("c2", "scen.csv"), net.n)
    res = oc.run(net, inj, 3e-3)
    _check_trace("c2", "mag_3e-3", res)


REF_BIN = oc.ROOT / "oracle" / "_ref" / "kronred_ref"

GEN_CASES = [
    dict(n=40, seed=6, slack=17),
    dict(n=80, seed=4, zfrac=0.3, shunts=True, lateral=0.6),
    dict(n=120, seed=8, lateral=0.5),
    dict(n=3, seed=9),
]


def _ref_trace(netp, scp, tmp, e_bar, obj, target):
    import subprocess

    tr = tmp / "trace.txt"
    cmd = [str(REF_BIN), "reduce", "--net", str(netp), "--scen", str(scp), "--e-bar", repr(e_bar),
           "--objective", obj, "--trace-hex", str(tr), "--workers", "1"]
    if target is not None:
        cmd += ["--target", repr(target)]
    subprocess.run(cmd, check=True, capture_output=True)
    rows, final = [], []
    for line in tr.read_text().splitlines():
        f = line.split()
        if f[0] == "final":
            final = f[1:]
        else:
            rows.append((int(f[1]), int(f[2]), f[3], f[4:-2], int(f[-2]), int(f[-1])))
    return rows, final


@pytest.mark.skipif(not REF_BIN.exists(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("kw", GEN_CASES, ids=lambda k: f"n{k['n']}s{k['seed']}")
@pytest.mark.parametrize("e_bar,obj,target", [(2e-3, "magnitude", None), (5e-3, "complex", None),
                                              (1e-2, "magnitude", 0.4), (0.0, "magnitude", None)])
def test_oracle_matches_reference_on_generated_feeders(kw, e_bar, obj, target, tmp_path):
    """Same check against the reference binary run here, on seeded feeders with
    unbalanced laterals, z_block branches, shunts and an off-zero slack."""
    import netgen

    netp, scp = netgen.write_case(tmp_path, L=3, **kw)
    rows, final = _ref_trace(netp, scp, tmp_path, e_bar, obj, target)
    net = oc.OracleNet(netp)
    res = oc.run(net, oc.read_currents(scp, net.n), e_bar, obj, target)
    assert len(rows) == len(res["s"])
    for i, (s, r, smice, errs, nsup, ncand) in enumerate(rows):
        assert (s, r, smice) == (res["s"][i], res["r"][i], gi.d2h(res["smice"][i]))
        assert errs == _hex(res["max_err"][i])
        assert (nsup, ncand) == (res["nsup"][i], res["cands"][i])
    assert final == _hex(res["final"])
