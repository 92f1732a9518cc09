"""In-tree build of libp2bw.so (the B200 engine + C-ABI) for sm_100a.

Every ``csrc/*.cu`` / ``csrc/*.cpp`` is compiled with nvcc
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``) into ``build/`` and
linked into ``paper_2006_09503_b200/libp2bw.so``.  Objects are rebuilt when the
source or any header in ``csrc/`` or ``include/`` is newer.  nvcc
cross-compiles without a GPU, so this runs in the CPU container as well.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "p2bw"
LIB = PKG / "libp2bw.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def find_json_include() -> str:
    """Directory holding nlohmann/json.hpp (header-only; the JSON library the reference's
    profile / plan I/O uses, profile.cpp:6).  P2BW_JSON_INCLUDE wins; otherwise the usual
    system prefixes and the copies Python packages vendor (cudnn-frontend ships one)."""
    env = os.environ.get("P2BW_JSON_INCLUDE")
    cands = [env] if env else []
    cands += ["/usr/include", "/usr/local/include"]
    for sp in sys.path:
        if sp and os.path.isdir(sp):
            cands += [os.path.join(sp, "include", "cudnn_frontend", "thirdparty"),
                      os.path.join(sp, "nvidia", "cudnn", "include")]
    cands += [os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                           "site-packages", "include", "cudnn_frontend", "thirdparty")]
    for c in cands:
        if c and os.path.isfile(os.path.join(c, "nlohmann", "json.hpp")):
            return c
    raise RuntimeError("nlohmann/json.hpp not found: install nlohmann-json (header-only) or point "
                       "P2BW_JSON_INCLUDE at the directory that contains nlohmann/json.hpp")


def _common() -> list[str]:
    return ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
            f"-I{CSRC}", f"-I{INCLUDE}", f"-I{find_json_include()}"]


def _sources() -> list[Path]:
    return sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.cpp")])


def _headers_mtime() -> float:
    hs = [*CSRC.glob("*.h"), *CSRC.glob("*.cuh"), *INCLUDE.rglob("*.h"), *INCLUDE.rglob("*.hpp")]
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    cmd = [NVCC, *ARCH, *_common(), "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    hdr = _headers_mtime()
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(tmp), *map(str, objs),
           "-lcudart_static", "-ldl", "-lpthread", "-lrt"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
