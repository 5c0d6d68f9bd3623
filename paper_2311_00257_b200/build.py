"""In-tree native build of libamsp.so (planner + C-ABI + sm_100a engine) and
of the CPU oracle (test infrastructure).

No JIT cache, no setuptools: objects go to paper_2311_00257_b200/_build/ and
the shared library to paper_2311_00257_b200/libamsp.so, so the built files
travel with the repo snapshot to the GPU box. Rebuilds are incremental on
(source mtime, header mtimes, command line).
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import site
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
BUILD = PKG / "_build"
LIB = PKG / "libamsp.so"
ORACLE_DIR = REPO / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "libamsp_oracle.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
# The image exports CXX=/opt/gcc/bin/g++, a wrapper without libgomp.spec.
CXX = os.environ.get("AMSP_CXX", "/usr/bin/g++")
CC = os.environ.get("AMSP_CC", "/usr/bin/gcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _json_include() -> str:
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        p = Path(sp) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
        if (p / "json.hpp").exists():
            return str(p)
    raise RuntimeError("nlohmann/json.hpp (cudnn_frontend) not found in site-packages")


def _headers() -> list[Path]:
    hs = list((REPO / "include").rglob("*.h*")) + list((PKG / "csrc").rglob("*.h"))
    hs += list((PKG / "csrc").rglob("*.cuh"))
    return hs


def _stamp(cmd: list[str], src: Path, deps: list[Path]) -> str:
    h = hashlib.sha1(" ".join(cmd).encode())
    for p in [src, *deps]:
        h.update(f"{p}:{p.stat().st_mtime_ns}".encode())
    return h.hexdigest()


def _run(cmd: list[str], obj: Path, src: Path, deps: list[Path], log: list[str]) -> None:
    stamp_file = obj.with_suffix(obj.suffix + ".stamp")
    stamp = _stamp(cmd, src, deps)
    if obj.exists() and stamp_file.exists() and stamp_file.read_text() == stamp:
        return
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        log.append(f"[{src.name}]\n{r.stderr.strip()}")
    stamp_file.write_text(stamp)


def build_library(verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    inc = ["-I", str(REPO / "include"), "-I", str(PKG / "csrc"), "-I", _json_include()]
    cuda_inc = ["-I", str(CUDA_HOME / "include")]
    cxxflags = ["-std=c++20", "-O2", "-fPIC", "-fopenmp", "-Wall", "-Wno-unknown-pragmas"]
    deps = _headers()
    jobs: list[tuple[list[str], Path, Path]] = []
    objs: list[Path] = []
    for src in sorted((PKG / "csrc").rglob("*.cpp")):
        obj = BUILD / (src.relative_to(PKG / "csrc").as_posix().replace("/", "__") + ".o")
        cmd = [CXX, *cxxflags, *inc, *cuda_inc, "-c", str(src), "-o", str(obj)]
        jobs.append((cmd, obj, src))
        objs.append(obj)
    for src in sorted((PKG / "csrc").rglob("*.cu")):
        obj = BUILD / (src.relative_to(PKG / "csrc").as_posix().replace("/", "__") + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v", *inc, "-c", str(src), "-o", str(obj)]
        jobs.append((cmd, obj, src))
        objs.append(obj)
    log: list[str] = []
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        futs = [ex.submit(_run, c, o, s, deps, log) for c, o, s in jobs]
        for f in futs:
            f.result()
    if log:
        (BUILD / "compile.log").write_text("\n\n".join(log) + "\n")
        if verbose:
            print("\n\n".join(log))
    link = [CXX, "-shared", "-fopenmp", "-o", str(LIB) + ".tmp", *map(str, objs),
            "-L", str(CUDA_HOME / "lib64"), "-lcudart_static", "-ldl", "-lrt", "-lpthread",
            "-Wl,--no-undefined"]
    newest = max(o.stat().st_mtime_ns for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime_ns < newest:
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}\n{r.stderr}")
        os.replace(str(LIB) + ".tmp", LIB)
    return LIB


def build_oracle() -> Path:
    """CPU checker (test infrastructure; never on the product path)."""
    ORACLE_LIB.parent.mkdir(exist_ok=True)
    src = ORACLE_DIR / "amsp_oracle.c"
    cmd = [CC, "-std=c11", "-O2", "-fPIC", "-fopenmp", "-ffp-contract=off", "-shared",
           str(src), "-o", str(ORACLE_LIB), "-lm"]
    stamp_file = ORACLE_LIB.with_suffix(".stamp")
    stamp = _stamp(cmd, src, [ORACLE_DIR / "amsp_oracle.h"])
    if ORACLE_LIB.exists() and stamp_file.exists() and stamp_file.read_text() == stamp:
        return ORACLE_LIB
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stderr}")
    stamp_file.write_text(stamp)
    return ORACLE_LIB


def build_reference() -> None:
    """Compile the reference planner into oracle/_ref when it is mounted."""
    if Path("/root/reference/proj/src").is_dir():
        subprocess.run(["bash", str(ORACLE_DIR / "build_ref.sh")], check=True,
                       capture_output=True)


PLAN_TIME = BUILD / "plan_time"


def build_plan_time() -> Path:
    """tests/cpp/plan_time.cpp (planner/simulator timing through the public
    shardplan API) linked against libamsp.so; oracle/build_ref.sh links the
    same source against the reference."""
    src = REPO / "tests" / "cpp" / "plan_time.cpp"
    cmd = [CXX, "-std=c++20", "-O2", "-I", str(REPO / "include"), str(src), "-o",
           str(PLAN_TIME), "-L", str(PKG), "-lamsp", "-Wl,-rpath,$ORIGIN/.."]
    stamp_file = PLAN_TIME.with_suffix(".stamp")
    stamp = _stamp(cmd, src, _headers() + [LIB])
    if PLAN_TIME.exists() and stamp_file.exists() and stamp_file.read_text() == stamp:
        return PLAN_TIME
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"plan_time build failed:\n{r.stderr}")
    stamp_file.write_text(stamp)
    return PLAN_TIME


def build_all(verbose: bool = False) -> None:
    build_library(verbose)
    build_plan_time()
    build_oracle()
    build_reference()


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
    print(f"built {LIB} and {ORACLE_LIB}")
