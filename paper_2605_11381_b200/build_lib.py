"""Build libkairos_b200.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2605_11381_b200.build_lib [--force]

Every translation unit is compiled with -fmad=false: the fp64 arithmetic must
follow the reference's evaluation order exactly, with fused multiply-adds only
where the kernels request them explicitly (__fma_rn).
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
OUT = PKG / "libkairos_b200.so"
PACK_SRC = CSRC / "kr_pack.c"  # host runtime: CPython extension (object packing)
OBJ = PKG / "build"

SOURCES = ["kr_capi.cu", "kr_horizon.cu", "kr_div_skx.cu", "kr_div_hsw.cu", "kr_sweep.cu",
           "kr_sweep_f32.cu", "kr_sweep_f64.cu",
           "kr_urgency.cu", "kr_select.cu", "kr_synth.cu", "kr_ingest.cpp"]
HEADERS = ["kr_common.cuh", "kr_host.cuh", "kr_stream.cuh", "kr_plan.cuh", "kr_conf.cuh",
           "kr_sweep.cuh", "kr_div.cuh", "kr_select_state.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-Xptxas", "-warn-spills",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libkairos_b200.so")


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [INCLUDE / "kairos_b200.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def pack_module_path() -> Path:
    import sysconfig
    return PKG / ("_kr_pack" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pack(force: bool = False) -> Path:
    """The native object packer (_kr_pack, kr_pack.c) with the host C compiler."""
    import sysconfig
    out = pack_module_path()
    if not force and out.exists() and out.stat().st_mtime >= PACK_SRC.stat().st_mtime:
        return out
    cc = os.environ.get("CC") or shutil.which("gcc") or "cc"
    tmp = out.with_suffix(".tmp")
    subprocess.run([cc, "-O2", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"],
                    str(PACK_SRC), "-o", str(tmp)], check=True)
    os.replace(tmp, out)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    build_pack(force)
    if not force and not _stale():
        return OUT
    OBJ.mkdir(exist_ok=True)
    cc = nvcc()
    objs = []
    procs = []
    for src in SOURCES:
        obj = OBJ / (Path(src).stem + ".o")
        cmd = [cc, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(str(obj))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append(f"--- {src}\n{out.decode()}")
        elif verbose and out:
            print(out.decode())
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    tmp = OUT.with_suffix(".so.tmp")
    link = [cc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", str(tmp),
            "-lcudart"]
    subprocess.run(link, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
