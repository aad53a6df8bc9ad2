"""Build libslimpipe.so in-tree (paper_2504_14519_b200/lib/).

Host C++ (planning + runtime) is compiled with g++ -O2; CUDA sources with
nvcc for sm_100a only (``-gencode arch=compute_100a,code=sm_100a -lineinfo``).
cudart is linked statically (nvcc default); cuBLASLt and NCCL are linked by
soname so the process shares whichever copy torch already loaded.
Incremental: an object is rebuilt when its source or any header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "obj"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libslimpipe.so"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC / 'host'}", f"-I{CSRC / 'cuda'}", f"-I{CUDA / 'include'}"]
# nlohmann/json (header-only; the scenario / Gantt text in csrc/host): the copy
# the image ships with cudnn_frontend, the same header the reference includes.
_NLOHMANN = [Path(p) / "include" / "cudnn_frontend" / "thirdparty" for p in sys.path if p.endswith("site-packages")]
HOST_INCLUDES = [f"-isystem{p}" for p in _NLOHMANN if (p / "nlohmann" / "json.hpp").exists()][:1]


def _headers() -> list[Path]:
    return sorted((ROOT / "include").rglob("*.h*")) + sorted(CSRC.rglob("*.h*")) + sorted(CSRC.rglob("*.cuh"))


def _sources() -> list[Path]:
    return sorted(CSRC.rglob("*.cpp")) + sorted(CSRC.rglob("*.cu"))


def _obj(src: Path) -> Path:
    rel = src.relative_to(CSRC)
    return BUILD / (str(rel).replace(os.sep, "__") + ".o")


def _compile_cmd(src: Path, obj: Path) -> list[str]:
    if src.suffix == ".cu":
        return [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                "-Xptxas", "-warn-spills", *INCLUDES, "-c", str(src), "-o", str(obj)]
    return ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter", *INCLUDES,
            *HOST_INCLUDES, "-c", str(src), "-o", str(obj)]


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    hdr_mtime = max((h.stat().st_mtime for h in _headers()), default=0.0)
    srcs = _sources()
    todo = []
    for s in srcs:
        o = _obj(s)
        if not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, hdr_mtime):
            todo.append((s, o))

    def run(cmd: list[str]) -> None:
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip()):
            print(r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(lambda so: run(_compile_cmd(*so)), todo))
    objs = [str(_obj(s)) for s in srcs]
    lib_mtime = LIB.stat().st_mtime if LIB.exists() else -1.0
    if todo or lib_mtime < max(os.path.getmtime(o) for o in objs):
        run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-Xlinker", "-Bsymbolic", "-o", str(LIB), *objs,
             f"-L{CUDA / 'lib64'}", "-lcublasLt", "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-lpthread", "-ldl"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
