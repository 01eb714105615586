"""In-tree build of the native libraries (sm_100a only).

    python -m paper_2505_16175_b200.build          # or __graft_entry__.build()

Products (git-ignored, but they travel to the GPU box with the gpurun snapshot):
  paper_2505_16175_b200/lib/libqvk.so          CUDA kernels + the C ABI of include/qvk.h
  paper_2505_16175_b200/lib/libqv_prefill.so   drop-in qv:: API (reference prefill.hpp) over libqvk.so
                                               (built only where the reference headers are present)
Test infrastructure (never imported by the product):
  oracle/  via its Makefile;  tests/native/build/parity_driver
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2505_16175_b200"
CSRC = PKG / "csrc"
LIB = PKG / "lib"
OBJ = ROOT / "build" / "obj"
INCLUDE = ROOT / "include"
REF_INCLUDE = Path(os.environ.get("QV_REF_INCLUDE", "/root/reference/proj/include"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> Path:
    """The NCCL torch bundles (site-packages/nvidia/nccl): linking the same runtime keeps one NCCL per process."""
    for p in map(Path, sys.path):
        d = p / "nvidia" / "nccl"
        if (d / "include" / "nccl.h").exists() and (d / "lib" / "libnccl.so.2").exists():
            return d
    raise RuntimeError("nvidia/nccl (torch's NCCL) not found on sys.path")


NCCL = _nccl_dir()
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = GENCODE + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                     f"-I{INCLUDE}", f"-I{CSRC}", f"-I{NCCL / 'include'}", "-ccbin", "g++"] + os.environ.get("QVK_EXTRA_NVFLAGS", "").split()
CXX = "g++"  # /usr/bin/g++ (the image's CXX variable points at a toolchain without libgomp)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_qvk(force: bool = False) -> Path:
    LIB.mkdir(parents=True, exist_ok=True)
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [INCLUDE / "qvk.h"]
    srcs = sorted(CSRC.glob("*.cu"))
    jobs = []
    for s in srcs:
        o = OBJ / (s.stem + ".o")
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC] + NVFLAGS + ["-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(_run, jobs))
    out = LIB / "libqvk.so"
    objs = [OBJ / (s.stem + ".o") for s in srcs]
    if force or jobs or _stale(out, objs):
        _run([NVCC] + GENCODE + ["-shared", "-o", str(out)] + [str(o) for o in objs] + ["-lcudart", f"-L{NCCL / 'lib'}", "-l:libnccl.so.2",
                                                                       f"-Xlinker=-rpath={NCCL / 'lib'}"])
    return out


def build_shim(force: bool = False) -> Path | None:
    """The qv:: drop-in is compiled against the reference's own, unchanged headers (read in place)."""
    out = LIB / "libqv_prefill.so"
    if not (REF_INCLUDE / "qv" / "prefill.hpp").exists():
        return out if out.exists() else None
    src = CSRC / "shim" / "prefill_shim.cpp"
    if force or _stale(out, [src, INCLUDE / "qvk.h", LIB / "libqvk.so"]):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", f"-I{REF_INCLUDE}", f"-I{INCLUDE}",
              str(src), "-o", str(out), f"-L{LIB}", "-lqvk", "-Wl,-rpath,$ORIGIN"])
    return out


def build_pipeline(force: bool = False) -> Path | None:
    """The overlap pipeline (include/qv_pipeline.hpp) over the drop-in; its producer is the reference's unchanged
    video side, resolved at link time of the application (as qv::decode_intervals would be)."""
    out = LIB / "libqv_pipeline.so"
    if not (REF_INCLUDE / "qv" / "decode.hpp").exists():
        return out if out.exists() else None
    src = CSRC / "shim" / "pipeline.cpp"
    if force or _stale(out, [src, INCLUDE / "qv_pipeline.hpp", LIB / "libqv_prefill.so"]):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra", f"-I{REF_INCLUDE}",
              f"-I{INCLUDE}", str(src), "-o", str(out), f"-L{LIB}", "-lqv_prefill", "-Wl,-rpath,$ORIGIN"])
    return out


def build_oracle() -> None:
    """Test infrastructure: the reference (when /root/reference is present) and the C restatement."""
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


def build_native_tests(force: bool = False) -> Path | None:
    """Test infrastructure: C++ parity driver linking the drop-in (qv::) beside the reference oracle (qvref::)."""
    ref_lib = ROOT / "oracle" / "_ref"
    shim = LIB / "libqv_prefill.so"
    out = ROOT / "tests" / "native" / "build" / "parity_driver"
    src = ROOT / "tests" / "native" / "parity_driver.cpp"
    if not (REF_INCLUDE / "qv" / "prefill.hpp").exists() or not shim.exists():
        return out if out.exists() else None
    out.parent.mkdir(parents=True, exist_ok=True)
    if force or _stale(out, [src, shim, LIB / "libqv_pipeline.so"]):
        _run([CXX, "-std=c++20", "-O2", "-Wall", "-pthread", f"-I{REF_INCLUDE}", f"-I{INCLUDE}", str(src), "-o",
              str(out), f"-L{LIB}", "-lqv_pipeline", "-lqv_prefill", "-lqvk", f"-L{ref_lib}", "-lqv_video", "-lqvref_capi", "-lqvref",
              "-Wl,-rpath,$ORIGIN/../../../paper_2505_16175_b200/lib:$ORIGIN/../../../oracle/_ref", "-fopenmp"])
    return out


def build_all(force: bool = False) -> None:
    build_qvk(force)
    build_shim(force)
    build_pipeline(force)
    build_oracle()
    build_native_tests(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", ", ".join(str(p.relative_to(ROOT)) for p in sorted(LIB.glob("*.so"))))
