"""Build the native library libtofr_b200.so in-tree (sm_100a, no JIT).

Device code: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo
--fmad=false (FP64 parity path: the reference is an x86-64 build without FMA
contraction, so no fused multiply-adds keeps the arithmetic identical).
Host runtime: g++ -O2 -ffp-contract=off (the BVH build and beam trace must
match the reference host arithmetic).  The CUDA runtime is linked statically
so the .so only needs the driver on the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OUT_DIR = PKG / "_native"
BUILD_DIR = PKG.parent / "build" / "native"
LIB = OUT_DIR / "libtofr_b200.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"

DEVICE_SOURCES = ["tofr_kernels.cu", "tofr_wave.cu", "tofr_trace.cu", "bvh_build.cu"]
HOST_SOURCES = ["host_scene.cpp", "capi.cpp", "ktime.cpp", "halo_transport.cpp"]
HEADERS = [
    "tofr_core.h",
    "tofr_geom.h",
    "tofr_path.cuh",
    "tofr_ellipsoid.cuh",
    "tofr_store.cuh",
    "tofr_kcommon.cuh",
    "ktime.h",
    "tofr_kernels.h",
    "host_scene.h",
    "halo_transport.h",
    "bvh_build.h",
]


def _cxx() -> str:
    return shutil.which("g++") or "g++"


def _newest_input() -> float:
    files = [CSRC / f for f in DEVICE_SOURCES + HOST_SOURCES + HEADERS]
    files.append(INCLUDE / "tofr_gpu.h")
    files.append(Path(__file__))
    return max(f.stat().st_mtime for f in files)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")


def needs_build() -> bool:
    return not LIB.exists() or LIB.stat().st_mtime < _newest_input()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA/C++ source of the package for sm_100a."""
    if not force and not needs_build():
        return LIB
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    BUILD_DIR.mkdir(parents=True, exist_ok=True)
    objs = []
    procs = []
    for src in DEVICE_SOURCES:
        obj = BUILD_DIR / (src + ".o")
        cmd = [NVCC, "-std=c++17", GENCODE, "-O3", "-lineinfo", "--fmad=false",
               "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", str(CSRC), "-I", str(INCLUDE),
               "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for src in HOST_SOURCES:
        obj = BUILD_DIR / (src + ".o")
        cmd = [_cxx(), "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-I", str(CSRC),
               "-I", str(INCLUDE), "-I", str(CUDA_HOME / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    failed = False
    for cmd, p in procs:
        out, err = p.communicate()
        if verbose:
            print(" ".join(cmd), flush=True)
        if p.returncode != 0:
            sys.stderr.write(out + err)
            failed = True
    if failed:
        raise RuntimeError("native build failed")
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, GENCODE, "-shared", "-cudart", "static", "-o", str(tmp)] + [str(o) for o in objs]
         + ["-ldl", "-Xlinker", "-rpath,$ORIGIN"], verbose)
    os.replace(tmp, LIB)
    return LIB


def build_variants(variants: dict, verbose: bool = False) -> dict:
    """Tuning builds: {tag: [-D...]} -> _native/variants/libtofr_b200_<tag>.so
    (same host objects as the main library; only the device code differs).
    Select one at run time with TOFR_B200_LIB=<path>."""
    build(verbose=verbose)
    vdir = OUT_DIR / "variants"
    vdir.mkdir(parents=True, exist_ok=True)
    host_objs = [BUILD_DIR / (src + ".o") for src in HOST_SOURCES]
    procs, outs = [], {}
    for tag, defs in variants.items():
        objs = []
        for src in DEVICE_SOURCES:
            obj = BUILD_DIR / f"{Path(src).stem}_{tag}.o"
            cmd = [NVCC, "-std=c++17", GENCODE, "-O3", "-lineinfo", "--fmad=false", *defs,
                   "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", str(CSRC), "-I", str(INCLUDE),
                   "-c", str(CSRC / src), "-o", str(obj)]
            procs.append((tag, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
            objs.append(obj)
        outs[tag] = objs
    for tag, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"variant {tag} failed")
    libs = {}
    for tag, objs in outs.items():
        lib = vdir / f"libtofr_b200_{tag}.so"
        _run([NVCC, GENCODE, "-shared", "-cudart", "static", "-o", str(lib)] + [str(o) for o in objs]
             + [str(o) for o in host_objs] + ["-ldl", "-Xlinker", "-rpath,$ORIGIN"], verbose)
        libs[tag] = lib
    return libs


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
