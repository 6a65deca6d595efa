"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
and the host half of the path (parsing, validation, enumeration/commit state
machine, sharding, min-loc merge) reproduces the reference's behaviour."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2510_19608_b200 as kr
from golden_io import path, read_trace, runs

ROOT = Path(__file__).resolve().parents[1]


def header_symbols() -> list[str]:
    text = (ROOT / "include" / "kronred_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(krg_[a-z_0-9]+)\s*\(", text)) - {"krg_exchange_fn", "krg_observer_fn"})


def test_library_exports_every_header_symbol():
    lib = kr.lib()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(kr.api.exported_symbols()) <= set(header_symbols())
    assert b"sm_100a" in lib.krg_version()


def test_host_parse_matches_reference_json():
    import json
    hp = kr.HostProblem(str(path("c1", "net.json")), str(path("c1", "scen.csv")))
    j = json.loads(path("c1", "net.json").read_text())
    assert hp.network.size == len(j["nodes"]) == 100
    assert hp.network.slack == 0
    assert len(hp.library.ids) == 4 and not hp.library.pq
    b0 = j["branches"][0]
    yb = np.array(b0["y_block"])
    np.testing.assert_array_equal(hp.network.y_series[0].real, yb[:, 0])
    np.testing.assert_array_equal(hp.network.y_series[0].imag, yb[:, 1])
    hp2 = kr.HostProblem(str(path("pq30", "net.json")), str(path("pq30", "scen_pq.csv")))
    assert hp2.library.pq and hp2.library.ids == ["s0", "s1", "s2"]


@pytest.mark.parametrize("case,tag", [("c1", "mag_1e-3"), ("c1", "complex_1e-3"), ("m40", "mag_1e-2"),
                                      ("c2", "mag_3e-3")])
def test_enumeration_follows_reference_trajectory(case, tag):
    hp = kr.HostProblem(str(path(case, "net.json")))
    rows, _ = read_trace(case, tag)
    traj = []
    step = max(1, len(rows) // 25)
    for i, (s, r, _sm, _me, snc, cc) in enumerate(rows):
        if i % step == 0:
            cands = kr.enumerate_after(hp.network, traj)
            assert len(cands) == cc, (i, len(cands), cc)
            assert (s, r) in cands
            assert cands == sorted(cands)
        traj.append((s, r))
    assert len(kr.enumerate_after(hp.network, traj)) >= 0


def test_commit_rejects_structural_misuse():
    hp = kr.HostProblem(str(path("s24", "net.json")))
    with pytest.raises(kr.Error):
        kr.enumerate_after(hp.network, [(1, 0)])  # slack as r
    with pytest.raises(kr.Error):
        kr.enumerate_after(hp.network, [(0, 23)])  # not adjacent


def test_validation_errors():
    hp = kr.HostProblem(str(path("s24", "net.json")))
    net = hp.network
    kr.validate(net)
    bad = kr.Network(net.phases.copy(), net.slack, net.slack_voltage, net.br_from.copy(), net.br_to.copy(),
                     net.y_series, net.shunt_from, net.shunt_to)
    bad.br_to[3] = bad.br_from[3]  # self loop
    with pytest.raises(kr.ValidationError):
        kr.validate(bad)
    bad2 = kr.Network(net.phases.copy(), 5, net.slack_voltage, net.br_from, net.br_to, net.y_series)
    with pytest.raises(kr.ValidationError):
        kr.validate(bad2)


def test_scenario_csv_errors(tmp_path):
    net = str(path("s24", "net.json"))
    p = tmp_path / "bad.csv"
    p.write_text("scenario_id,node_id,phase,x,y\n")
    with pytest.raises(kr.ValidationError):
        kr.HostProblem(net, str(p))
    p.write_text("scenario_id,node_id,phase,i_re,i_im\ns0,1,z,0,0\n")
    with pytest.raises(kr.ValidationError):
        kr.HostProblem(net, str(p))
    p.write_text("scenario_id,node_id,phase,i_re,i_im\ns0,999,a,0,0\n")
    with pytest.raises(kr.ValidationError):
        kr.HostProblem(net, str(p))
    p.write_text("")
    assert kr.HostProblem(net, str(p)).library.ids == []


def test_shard_range_partitions_contiguously():
    for count in [0, 1, 7, 100, 16759]:
        for world in [1, 2, 3, 8]:
            spans = [kr.shard_range(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_merge_best_lexicographic():
    assert kr.merge_best([1.0, 0.5, 0.5], [3, 9, 7]) == 2
    assert kr.merge_best([np.inf, 2.0], [-1, 4]) == 1
    assert kr.merge_best([1.0, 1.0], [-1, -1]) == -1


def test_device_entry_fails_loudly_without_gpu():
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    hp = kr.HostProblem(str(path("s24", "net.json")), str(path("s24", "scen.csv")))
    with pytest.raises(kr.CudaError):
        kr.Context(hp)


def test_golden_runs_are_consistent():
    # fixture sanity: every committed trace has supernode counts decreasing by one
    for case in ["c1", "m40", "s24", "r30"]:
        for tag in runs(case):
            rows, final = read_trace(case, tag)
            n = kr.HostProblem(str(path(case, "net.json"))).network.size
            for i, row in enumerate(rows):
                assert row[4] == n - 1 - i


def _build_dropin(tmp_path):
    import subprocess
    exe = tmp_path / "dropin_reduce"
    lib = ROOT / "paper_2510_19608_b200" / "_lib"
    kr.lib()  # builds the library if needed
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tools" / "dropin_reduce.cpp"),
                    f"-L{lib}", "-lkronred_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    return exe


def test_cpp_dropin_compiles_against_header(tmp_path):
    """tools/dropin_reduce.cpp is the reference CLI's cmd_reduce (main.cpp:52-120)
    with only the include swapped; it must compile and link against the .so."""
    exe = _build_dropin(tmp_path)
    assert exe.exists()
