"""Build libkronred_b200.so in-tree (sm_100a) — nvcc for the CUDA engine,
g++ for the host C++; the shared object travels with the repo snapshot."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib"
LIB = OUT / "libkronred_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL 2.28 (host + device API: symmetric windows, LSA barriers) for the
# in-graph multi-GPU min-loc exchange; the torch-bundled build of this image
NCCL = Path(os.environ.get("KRONRED_NCCL", "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"))
COMMON = ["-O3", "-std=c++20", f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{NCCL / 'include'}"]
NCCL_LINK = [f"-L{NCCL / 'lib'}", "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", str(NCCL / "lib")]
NVFLAGS = COMMON + ARCH + ["-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
                           "-Xptxas", "-v", "--expt-relaxed-constexpr"]
CXXFLAGS = COMMON + ["-fPIC", "-ffp-contract=off", "-Wall", "-Wextra", "-I/usr/local/cuda/include"]


def _run(cmd: list[str]) -> str:
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return p.stdout + p.stderr


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cpp")) + sorted(CSRC.glob("*.cu"))


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list((ROOT / "include").glob("*")) + [Path(__file__)]
    return all(d.stat().st_mtime <= t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    OUT.mkdir(exist_ok=True)
    objs, jobs = [], []
    for src in sources():
        obj = OUT / (src.name + ".o")
        objs.append(obj)
        if src.suffix == ".cu":
            cmd = [NVCC, *NVFLAGS, "-c", str(src), "-o", str(obj)]
        else:
            cmd = [CXX, *CXXFLAGS, "-c", str(src), "-o", str(obj)]
        jobs.append(cmd)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        logs = list(ex.map(_run, jobs))
    (OUT / "ptxas.log").write_text("\n".join(l for l in logs if l))
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, "-shared", *ARCH, "-o", str(tmp), *map(str, objs), *NCCL_LINK, "-lcudart_static", "-lrt", "-ldl",
          "-lpthread"])
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_variant(out_dir: Path, defines: list[str]) -> Path:
    """Tuning aid: the library with the CUDA engine recompiled under extra
    -D defines, into out_dir (host objects reused from the main build).
    Load it with KRONRED_LIB=<out_dir>/libkronred_b200.so."""
    build()
    out_dir.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in sources():
        if src.suffix == ".cu":
            obj = out_dir / (src.name + ".o")
            _run([NVCC, *NVFLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)])
        else:
            obj = OUT / (src.name + ".o")
        objs.append(obj)
    lib = out_dir / LIB.name
    _run([NVCC, "-shared", *ARCH, "-o", str(lib), *map(str, objs), *NCCL_LINK, "-lcudart_static", "-lrt", "-ldl",
          "-lpthread"])
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:  # build.py --variant DIR [DEFINE ...]
        i = sys.argv.index("--variant")
        print(build_variant(Path(sys.argv[i + 1]), sys.argv[i + 2:]))
    else:
        build(force="--force" in sys.argv, verbose=True)
