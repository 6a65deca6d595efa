"""Regenerate the golden fixtures under tests/golden from the reference build.

Runs oracle/_ref/kronred_ref (the UNMODIFIED reference library compiled by
oracle/Makefile from /root/reference/proj/src) and stores its inputs/outputs:

  <case>/net.json, scen.csv        inputs (reference writer; current-mode CSV
                                   whose reload is bit-identical, checked by `gen`)
  <case>/trace_<tag>.txt           committed (s, r, smice, max_err[]) as IEEE hex
  <case>/reduced_<tag>.json        reference reduced-model JSON (byte target)
  <case>/scores_<tag>.txt          per-candidate delta scores, first iterations
  <case>/solve.txt                 v0, V-hat, every unit-injection solve (hex)
  <case>/kron_<k>.txt + .reduce    kron_reduce blocks (hex) for random partitions

Usage: python tests/golden/make_golden.py   (needs /root/reference; run here,
never on the GPU box). Large inputs are gzipped.
"""
from __future__ import annotations

import gzip
import json
import random
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = ROOT / "oracle" / "_ref" / "kronred_ref"


def run(*args: str) -> str:
    p = subprocess.run([str(REF), *args], capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"{args}: {p.stderr}")
    return p.stdout


def gen(case: str, **kw) -> Path:
    d = HERE / case
    d.mkdir(exist_ok=True)
    args = ["gen", "--net", str(d / "net.json"), "--scen", str(d / "scen.csv")]
    for k, v in kw.items():
        if k == "pq":
            pass
        args += [f"--{k}", str(v)]
    out = json.loads(run(*args))
    assert out["roundtrip_bitwise"], case
    (d / "params.json").write_text(json.dumps(kw, indent=1) + "\n")
    return d


def reduce(d: Path, tag: str, *flags: str, radialize: bool = False, reduced: bool = True) -> dict:
    args = ["reduce", "--net", str(d / "net.json"), "--scen", str(d / "scen.csv"),
            "--trace-hex", str(d / f"trace_{tag}.txt"), *flags]
    if reduced:
        args += ["--reduced", str(d / f"reduced_{tag}.json")]
    if radialize:
        args.append("--radialize")
    out = json.loads(run(*args))
    meta = d / "runs.json"
    runs = json.loads(meta.read_text()) if meta.exists() else {}
    runs[tag] = {"flags": list(flags), "radialize": radialize, "iterations": out["iterations"],
                 "candidates": out["candidates"], "kept": out["kept"]}
    meta.write_text(json.dumps(runs, indent=1, sort_keys=True) + "\n")
    return out


def scores(d: Path, tag: str, iters: int, *flags: str) -> None:
    run("scores", "--net", str(d / "net.json"), "--scen", str(d / "scen.csv"), "--iters", str(iters),
        "--out", str(d / f"scores_{tag}.txt"), *flags)


def kron(d: Path, k: int, reduce_set: list[int]) -> None:
    (d / f"kron_{k}.reduce").write_text(" ".join(map(str, reduce_set)) + "\n")
    run("kron", "--net", str(d / "net.json"), "--reduce", str(d / f"kron_{k}.reduce"),
        "--out", str(d / f"kron_{k}.txt"))


def gz(path: Path) -> None:
    with open(path, "rb") as f, gzip.open(str(path) + ".gz", "wb", compresslevel=9) as g:
        shutil.copyfileobj(f, g)
    path.unlink()


def large() -> None:
    """BASELINE configs[2]/[3] shaped feeders (defaults, branching 0.3): the
    5,991-node and 8,381-node synthetic feeders with 2 scenarios, and the
    reference's first iterations (target = K/n; the CPU reference needs about
    10 s per feeder for its serial column build)."""
    for case, n, k in (("c3", 5991, 4), ("c4", 8381, 3)):
        d = gen(case, n=n, seed=n, L=2, branching=0.3)
        reduce(d, f"mag_3e-3_k{k}", "--e-bar", "3e-3", "--target", repr(k / n + 1e-12), "--workers", "0",
               reduced=False)
        for f in ["net.json", "scen.csv"]:
            gz(d / f)


def _inflate(case: str, name: str) -> Path:
    """Plain copy of a gzipped fixture input (the reference reads plain files)."""
    import gzip as _gz
    import tempfile
    src = HERE / case / (name + ".gz")
    dst = Path(tempfile.gettempdir()) / "kronred_long" / case / name
    dst.parent.mkdir(parents=True, exist_ok=True)
    with _gz.open(src, "rb") as f, open(dst, "wb") as g:
        shutil.copyfileobj(f, g)
    return dst


def _reduce_files(case: str, tag: str, net: Path, scen: Path, *flags: str, reduced: bool) -> dict:
    d = HERE / case
    d.mkdir(exist_ok=True)
    args = ["reduce", "--net", str(net), "--scen", str(scen), "--trace-hex", str(d / f"trace_{tag}.txt"),
            *flags]
    if reduced:
        args += ["--reduced", str(d / f"reduced_{tag}.json")]
    out = json.loads(run(*args))
    meta = d / "runs.json"
    runs = json.loads(meta.read_text()) if meta.exists() else {}
    runs[tag] = {"flags": list(flags), "radialize": False, "iterations": out["iterations"],
                 "candidates": out["candidates"], "kept": out["kept"], "ref_wall_s": out["wall_s"],
                 "ref_workers": out["workers"]}
    meta.write_text(json.dumps(runs, indent=1, sort_keys=True) + "\n")
    gz(d / f"trace_{tag}.txt")
    if reduced:
        gz(d / f"reduced_{tag}.json")
    return out


def long(which: list[str]) -> None:
    """Whole-run / long-prefix goldens for BASELINE configs[2..4] (VERDICT r1
    item 1). Each step is independent; run in the background (hours of CPU):

      h2k   2,000-node three-phase-heavy feeder (frac2=0.003, frac1=0.005),
            5 scenarios, e_bar 3e-3, full run + first-2-iteration scores
      c3    5,991 nodes, 2 scenarios, e_bar 3e-3, target 0.9 (full run)
      c4L24 8,381 nodes, 24 scenarios, first 200 iterations
      c5    8,381 nodes, 96 scenarios, e_bar 1e-3, first 50 iterations
      c4    8,381 nodes, 2 scenarios, e_bar 3e-3, target 0.8 (full run)

    c4L24 / c5 libraries are too large to commit; the GPU tests regenerate
    them with the reference generator in oracle/_ref (params.json)."""
    import tempfile
    tmp = Path(tempfile.gettempdir()) / "kronred_long"
    tmp.mkdir(exist_ok=True)
    for w in which:
        if w == "h2k":
            d = gen("h2k", n=2000, seed=2000, L=5, branching=0.3, frac2=0.003, frac1=0.005)
            reduce(d, "mag_3e-3", "--e-bar", "3e-3", "--workers", "0")
            scores(d, "mag_3e-3", 2, "--e-bar", "3e-3")
            for f in ["net.json", "scen.csv", "trace_mag_3e-3.txt", "reduced_mag_3e-3.json", "scores_mag_3e-3.txt"]:
                gz(d / f)
        elif w == "c3":
            _reduce_files("c3", "mag_3e-3_t09", _inflate("c3", "net.json"), _inflate("c3", "scen.csv"),
                          "--e-bar", "3e-3", "--target", "0.9", "--workers", "0", reduced=True)
        elif w == "c4":
            _reduce_files("c4", "mag_3e-3_t08", _inflate("c4", "net.json"), _inflate("c4", "scen.csv"),
                          "--e-bar", "3e-3", "--target", "0.8", "--workers", "0", reduced=True)
        elif w in ("c4L24", "c5"):
            L, e, k = (24, "3e-3", 200) if w == "c4L24" else (96, "1e-3", 50)
            d = HERE / w
            d.mkdir(exist_ok=True)
            params = {"n": 8381, "seed": 8381, "L": L, "branching": 0.3}
            (d / "params.json").write_text(json.dumps(params, indent=1) + "\n")
            net, scen = tmp / f"{w}_net.json", tmp / f"{w}_scen.csv"
            run("gen", "--n", "8381", "--seed", "8381", "--L", str(L), "--branching", "0.3",
                "--net", str(net), "--scen", str(scen))
            assert net.read_bytes() == _inflate("c4", "net.json").read_bytes()
            _reduce_files(w, f"mag_{e}_k{k}", net, scen, "--e-bar", e, "--target", repr(k / 8381 + 1e-12),
                          "--workers", "0", reduced=False)
        else:
            raise SystemExit(f"unknown long step {w}")


def traces() -> None:
    """Trace CSV (io.cpp:338-359, wall_ms zeroed) and validate report
    (io.cpp:385-416, 20 bins) bytes of reference runs, for the writers'
    byte-level parity (run separately: `make_golden.py traces`)."""
    jobs = [("c1", "mag_1e-3", "scen.csv", ["--e-bar", "1e-3"], False),
            ("c1", "rad_1e-2_t06", "scen.csv", ["--e-bar", "1e-2", "--target", "0.6"], True),
            ("m40", "mag_1e-3", "scen.csv", ["--e-bar", "1e-3"], False),
            ("pq30", "pq_1e-3", "scen_pq.csv", ["--e-bar", "1e-3"], False),
            ("c2", "mag_3e-3", "scen.csv", ["--e-bar", "3e-3", "--workers", "0"], False)]
    for case, tag, scen, flags, rad in jobs:
        d = HERE / case
        net = _inflate(case, "net.json") if (d / "net.json.gz").exists() else d / "net.json"
        sc = _inflate(case, scen) if (d / (scen + ".gz")).exists() else d / scen
        args = ["reduce", "--net", str(net), "--scen", str(sc), *flags, "--trace", str(d / f"tracecsv_{tag}.csv"),
                "--validate", str(d / f"validate_{tag}.csv"), "--bins", "20"]
        if rad:
            args.append("--radialize")
        run(*args)
        if case == "c2":
            gz(d / f"tracecsv_{tag}.csv")


def naive() -> None:
    """use_delta = false (eval_full_solve, reduce.cpp:132-167) on the small
    feeders: its full solves round differently from the delta path."""
    reduce(HERE / "c1", "naive_mag_1e-3", "--e-bar", "1e-3", "--use-delta", "0")
    reduce(HERE / "c1", "naive_complex_1e-3", "--e-bar", "1e-3", "--objective", "complex", "--use-delta", "0")
    reduce(HERE / "m40", "naive_mag_1e-3", "--e-bar", "1e-3", "--use-delta", "0")
    reduce(HERE / "s24", "naive_mag_5e-4", "--e-bar", "5e-4", "--use-delta", "0")


def main() -> None:
    if not REF.exists():
        sys.exit("build oracle/_ref first: make -C oracle")
    if sys.argv[1:] == ["large"]:
        large()
        return
    if sys.argv[1:2] == ["long"]:
        long(sys.argv[2:] or ["h2k", "c3", "c4L24", "c5", "c4"])
        return
    if sys.argv[1:] == ["traces"]:
        traces()
        return
    if sys.argv[1:] == ["naive"]:
        naive()
        return
    # C1: ~100-node acceptance-recipe feeder, 4 scenarios (BASELINE configs[0])
    d = gen("c1", n=100, seed=1000, L=4, preset="acceptance")
    for e in ["1e-4", "1e-3", "3e-3", "1e-2"]:
        reduce(d, f"mag_{e}", "--e-bar", e)
    reduce(d, "complex_1e-3", "--e-bar", "1e-3", "--objective", "complex")
    reduce(d, "mag_3e-3_t05", "--e-bar", "3e-3", "--target", "0.5")
    reduce(d, "rad_1e-2_t06", "--e-bar", "1e-2", "--target", "0.6", radialize=True)
    scores(d, "mag_1e-3", 3, "--e-bar", "1e-3")
    scores(d, "complex_1e-3", 2, "--e-bar", "1e-3", "--objective", "complex")
    rng = random.Random(1)
    for k in range(3):
        kron(d, k, sorted(i for i in range(1, 100) if rng.random() < 0.3 + 0.2 * k))
    # small default-recipe feeder: solver bit checks (every unit column)
    d = gen("s24", n=24, seed=101, L=2)
    run("solve", "--net", str(d / "net.json"), "--scen", str(d / "scen.csv"), "--out", str(d / "solve.txt"))
    reduce(d, "mag_5e-4", "--e-bar", "5e-4")
    reduce(d, "inf", "--e-bar", "inf")
    # three-phase-heavy feeder: full 3x3 blocks everywhere
    d = gen("m40", n=40, seed=77, L=3, frac2=0.003, frac1=0.005)
    run("solve", "--net", str(d / "net.json"), "--scen", str(d / "scen.csv"), "--out", str(d / "solve.txt"))
    for e in ["1e-4", "1e-3", "1e-2"]:
        reduce(d, f"mag_{e}", "--e-bar", e)
    reduce(d, "complex_1e-3", "--e-bar", "1e-3", "--objective", "complex")
    scores(d, "mag_1e-3", 4, "--e-bar", "1e-3")
    rng = random.Random(2)
    for k in range(3):
        kron(d, k, sorted(i for i in range(1, 40) if rng.random() < 0.4))
    # meshed mid-run reduction for radialization (acceptance criterion 7 style)
    d = gen("r30", n=30, seed=7003, L=2, branching=0.5)
    reduce(d, "rad_5e-3_t055", "--e-bar", "5e-3", "--target", "0.55", radialize=True)
    reduce(d, "mag_5e-3_t055", "--e-bar", "5e-3", "--target", "0.55")
    # constant-PQ scenario CSV (reference default writer)
    d = gen("pq30", n=30, seed=5, L=3, pq=str(HERE / "pq30" / "scen_pq.csv"))
    run("reduce", "--net", str(d / "net.json"), "--scen", str(d / "scen_pq.csv"), "--e-bar", "1e-3",
        "--trace-hex", str(d / "trace_pq_1e-3.txt"), "--reduced", str(d / "reduced_pq_1e-3.json"))
    run("solve", "--net", str(d / "net.json"), "--scen", str(d / "scen_pq.csv"), "--out", str(d / "solve_pq.txt"))
    # C2: the 1000-node, 24-scenario benchmark feeder (BASELINE configs[1])
    d = gen("c2", n=1000, seed=1000, L=24, preset="acceptance")
    reduce(d, "mag_3e-3", "--e-bar", "3e-3", "--workers", "0")
    reduce(d, "mag_1e-3", "--e-bar", "1e-3", "--workers", "0")
    scores(d, "mag_3e-3", 1, "--e-bar", "3e-3")
    for f in ["net.json", "scen.csv", "trace_mag_3e-3.txt", "trace_mag_1e-3.txt", "reduced_mag_3e-3.json",
              "reduced_mag_1e-3.json", "scores_mag_3e-3.txt"]:
        gz(d / f)


if __name__ == "__main__":
    main()
