"""In-tree build of libseqpipe_b200.so (host C++ planner + sm_100a CUDA + NCCL).

Objects are compiled in parallel with g++ (host planner, -ffp-contract=off so
the cwp double arithmetic is bit-identical to the reference) and nvcc
(-gencode arch=compute_100a,code=sm_100a -lineinfo). The shared library lands in
paper_2406_03488_b200/lib/ and travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "lib"
OBJ = PKG / "build_obj"
LIB = OUT / "libseqpipe_b200.so"
CLI_SRC = PKG / "cli" / "seqpipe_main.cpp"
CLI = PKG / "bin" / "seqpipe_b200"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")

def _nccl_dir() -> Path | None:
    """NCCL shipped with this image's torch wheel (2.28.x). Linking against it (not the
    older system libnccl) lets torch and this library share one libnccl.so.2 in a process."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        d = Path(list(spec.submodule_search_locations)[0])
        if (d / "lib" / "libnccl.so.2").exists():
            return d
    return None


NCCL = _nccl_dir()
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC}"] + ([f"-I{NCCL / 'include'}"] if NCCL else []) + \
    [f"-I{CUDA / 'include'}"]
NCCL_LINK = ([f"-L{NCCL / 'lib'}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{NCCL / 'lib'}"] if NCCL
             else ["-lnccl"])
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra", "-Wno-unused-parameter"]
NVFLAGS = [
    "-std=c++20", "-O3", "-Xcompiler", "-fPIC", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
]


def _sources():
    cpp = sorted(CSRC.rglob("*.cpp"))
    cu = sorted(CSRC.rglob("*.cu"))
    return cpp, cu


def _headers_digest() -> str:
    h = hashlib.sha1()
    for p in sorted(list((ROOT / "include").rglob("*.h*")) + list(CSRC.rglob("*.h*")) + list(CSRC.rglob("*.cuh"))):
        h.update(p.read_bytes())
    return h.hexdigest()[:12]


def _compile(src: Path, digest: str, verbose: bool) -> Path:
    rel = src.relative_to(CSRC)
    obj = OBJ / (str(rel).replace("/", "__") + ".o")
    stamp = obj.with_suffix(".stamp")
    key = hashlib.sha1(src.read_bytes()).hexdigest()[:12] + digest
    if obj.exists() and stamp.exists() and stamp.read_text() == key:
        return obj
    if src.suffix == ".cu":
        cmd = [NVCC, *NVFLAGS, *INCLUDES, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *CXXFLAGS, *INCLUDES, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    stamp.write_text(key)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    OUT.mkdir(exist_ok=True)
    OBJ.mkdir(exist_ok=True)
    cpp, cu = _sources()
    digest = _headers_digest()
    srcs = cu + cpp  # nvcc units first: they are the slow ones
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, digest, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not (LIB.exists() and LIB.stat().st_mtime >= newest):
        _link(objs, verbose)
    _build_cli(verbose)
    return LIB


def _link(objs, verbose: bool) -> None:
    cmd = [
        NVCC, "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
        *map(str, objs), "-o", str(LIB),
        f"-L{CUDA / 'lib64'}", "-lcudart", *NCCL_LINK, "-ldl",
        "-Xlinker", "-rpath,$ORIGIN",
    ]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")


def _build_cli(verbose: bool) -> None:
    """bin/seqpipe_b200: the command-line front end, linked against the library (rpath ../lib)."""
    CLI.parent.mkdir(exist_ok=True)
    if CLI.exists() and CLI.stat().st_mtime >= max(LIB.stat().st_mtime, CLI_SRC.stat().st_mtime):
        return
    cmd = ["g++", *[f for f in CXXFLAGS if f != "-fPIC"], *INCLUDES, str(CLI_SRC), "-o", str(CLI),
           f"-L{OUT}", "-lseqpipe_b200", "-Wl,-rpath,$ORIGIN/../lib", f"-L{CUDA / 'lib64'}", "-lcudart"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
