"""Build libmace_b200.so in-tree (nvcc, sm_100a).  Called by __graft_entry__.build()."""

from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.environ.get("MACE_LIB") or os.path.join(PKG, "libmace_b200.so")  # MACE_LIB: ablation builds
# (source, extra defines): k2_inst.cu is compiled once per super-voxel tile side
SV_SIDES = (2, 4, 6, 8, 12, 16)
# (each through a generated one-line wrapper k2_s<S>.cu, so every cubin carries its own name)
UNITS = [("mace.cu", []), ("cnn.cu", []), ("layout.cpp", []), ("sysmat.cpp", [])] + [
    (f"k2_s{s}.cu", [f"-DMACE_SV_SIDE={s}"]) for s in SV_SIDES]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "-Xptxas", "-v",
    "-I" + os.path.join(ROOT, "include"),
    "-shared",
    *os.environ.get("MACE_NVCC_EXTRA", "").split(),  # ablation builds (e.g. -DMACE_K2_MINB_W=12)
]


def _inputs():
    out = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".cpp", ".h"))]
    out.append(os.path.join(ROOT, "include", "mace_b200.h"))
    return out


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


def _compile(src, defs, obj):
    path = os.path.join(CSRC, src)
    if src.startswith("k2_s"):
        path = os.path.join(os.path.dirname(obj), src)
        with open(path, "w") as fh:
            fh.write('#include "k2_inst.cu"\n')
    cmd = [NVCC, *[f for f in FLAGS if f != "-shared"], "-I" + CSRC, *defs, "-c", "-o", obj, path]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return cmd, res


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every unit to an object in parallel (one nvcc per unit), then link the library."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    tag = f"{os.getpid()}"
    objdir = os.path.join(CSRC, f"_obj.tmp{tag}")
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    for src, defs in UNITS:
        stem = os.path.splitext(src)[0]
        jobs.append((src, defs, os.path.join(objdir, stem + ".o")))
    log = os.path.join(PKG, "csrc", "build.log")
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: _compile(*j), jobs))
    text = "".join(" ".join(cmd) + "\n" + res.stdout + res.stderr for cmd, res in results)
    failed = [res for _, res in results if res.returncode != 0]
    tmp = LIB + f".tmp{tag}"
    if not failed:
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
               *[j[2] for j in jobs], "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        text += " ".join(cmd) + "\n" + res.stdout + res.stderr
        if res.returncode != 0:
            failed.append(res)
    with open(log, "w") as fh:
        fh.write(text)
    import shutil

    shutil.rmtree(objdir, ignore_errors=True)
    if failed:
        raise RuntimeError(f"nvcc failed (see {log}):\n{failed[0].stderr[-4000:]}")
    os.replace(tmp, LIB)
    if verbose:
        print(text)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
