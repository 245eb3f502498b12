"""In-tree build of the sm_100a extension (libdopinf_b200.so) and the oracle.

The extension is compiled with nvcc for sm_100a only and linked against NCCL;
the .so lands next to this file so it travels to the GPU box with the repo
snapshot. The oracle (test infrastructure) is built by oracle/Makefile.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libdopinf_b200.so"
SOURCES = ["capi.cu", "capi_coll.cu", "gram_ref.cu", "capi_io.cu", "capi_post.cu", "gram.cu", "transform.cu", "project.cu", "synth.cu", "eig.cu", "field.cu", "rom.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-I", str(ROOT / "include"),
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the sm_100a extension cannot be built")


def _nccl_dir():
    """The NCCL torch ships (nvidia-nccl wheel), so one libnccl.so.2 serves both
    torch and this library in a process; the system copy only as a fallback."""
    try:
        import nvidia.nccl as n

        d = Path(list(n.__path__)[0])
        if (d / "lib" / "libnccl.so.2").exists() and (d / "include" / "nccl.h").exists():
            return d
    except Exception:  # noqa: BLE001
        pass
    return None


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_extension(force: bool = False, verbose: bool = False) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    nccl = _nccl_dir()
    flags = list(NVCC_FLAGS) + (["-I", str(nccl / "include")] if nccl else [])
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "dopinf_b200.h"]
    jobs = []
    for src in SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        if force or _stale(obj, [CSRC / src, *headers]):
            jobs.append([nvcc, *flags, "-c", str(CSRC / src), "-o", str(obj)])
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
            if verbose and (res.stdout or res.stderr):
                print(res.stdout, res.stderr)
    objs = [BUILD / (Path(s).stem + ".o") for s in SOURCES]
    if force or jobs or _stale(LIB, objs):
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(LIB),
               *map(str, objs)]
        if nccl:
            cmd += [f"-L{nccl / 'lib'}", "-l:libnccl.so.2", f"-Xlinker=-rpath,{nccl / 'lib'}"]
        else:
            cmd += ["-lnccl"]
        cmd += ["-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return LIB


def build_oracle(with_reference: bool | None = None) -> None:
    """oracle/_build (C restatement) always; oracle/_ref when /root/reference exists."""
    oracle = ROOT / "oracle"
    res = subprocess.run(["make", "-s", "-C", str(oracle), "oracle"], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")
    ref_src = Path(os.environ.get("DOPINF_REFERENCE", "/root/reference/proj"))
    if with_reference is None:
        with_reference = (ref_src / "src" / "pod.cpp").exists()
    if with_reference:
        res = subprocess.run(["make", "-s", "-j8", "-C", str(oracle), "ref", f"REF={ref_src}"],
                             capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"reference oracle build failed:\n{res.stdout}\n{res.stderr}")


def build_parity_harness() -> Path | None:
    """tests/cpp/_build/parity: the C++ drop-in compiled against the reference's
    headers and oracle/_ref/libdopinf_ref.a (test infrastructure; needs the
    reference sources, so it is built here and travels as a binary)."""
    ref_src = Path(os.environ.get("DOPINF_REFERENCE", "/root/reference/proj"))
    lib_ref = ROOT / "oracle" / "_ref" / "libdopinf_ref.a"
    if not (ref_src / "include" / "dopinf" / "pod.hpp").exists() or not lib_ref.exists():
        return None
    import scipy

    blas = Path(scipy.__file__).resolve().parent.parent / "scipy.libs"
    blas_lib = next(blas.glob("libscipy_openblas*.so"))
    out = ROOT / "tests" / "cpp" / "_build" / "parity"
    out.parent.mkdir(parents=True, exist_ok=True)
    src = ROOT / "tests" / "cpp" / "parity_main.cpp"
    if not _stale(out, [src, LIB, ROOT / "include" / "dopinf_b200.hpp", ROOT / "include" / "dopinf_b200_pipeline.hpp", lib_ref]):
        return out
    cmd = ["g++", "-std=gnu++20", "-O2", f"-I{ROOT / 'oracle' / 'shim'}", f"-I{ref_src / 'include'}",
           f"-I{ROOT / 'include'}", str(src), str(lib_ref), f"-L{PKG}", "-ldopinf_b200",
           "-Wl,-rpath,$ORIGIN/../../../paper_2504_14338_b200", f"-L{blas}", f"-l:{blas_lib.name}", f"-Wl,-rpath,{blas}", "-lpthread",
           "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"parity harness build failed:\n{res.stderr}")
    return out


def build_c_smoke() -> Path:
    """tests/c/_build/abi_smoke: the C ABI exercised from plain C11 (gcc)."""
    out = ROOT / "tests" / "c" / "_build" / "abi_smoke"
    out.parent.mkdir(parents=True, exist_ok=True)
    src = ROOT / "tests" / "c" / "abi_smoke.c"
    if not _stale(out, [src, LIB, ROOT / "include" / "dopinf_b200.h"]):
        return out
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", str(src), f"-L{PKG}",
           "-ldopinf_b200", "-Wl,-rpath,$ORIGIN/../../../paper_2504_14338_b200", "-lm", "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"C smoke build failed:\n{res.stderr}")
    return out


if __name__ == "__main__":
    print(build_extension(verbose=True))
    build_oracle()
    print(build_parity_harness())
    print(build_c_smoke())
